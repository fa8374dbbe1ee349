#!/usr/bin/env bash
# which weight-gradient GEMMs go to the side stream: CB_WGRAD_WAVE_EFF 0.9 (default) / 0.95 / 1.01 (all)
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for rep in a b; do
  for f in 0.9 0.95 1.01; do
    CB_WGRAD_WAVE_EFF=$f timeout 600 python bench.py --config 7b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/wave_7b_${f}_${rep}.log 2>&1
  done
done
for f in 0.9 0.95 1.01; do
  CB_WGRAD_WAVE_EFF=$f timeout 600 python bench.py --config 1b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/wave_1b_${f}.log 2>&1
done
