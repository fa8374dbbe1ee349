#!/usr/bin/env bash
# weight-gradient side stream on (CB_WGRAD_STREAM=4, default) vs off (0), with inline AdamW
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for rep in a b; do
  for f in 4 0; do
    CB_WGRAD_STREAM=$f timeout 600 python bench.py --config 7b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/wgs_7b_${f}_${rep}.log 2>&1
  done
done
for f in 4 0; do
  CB_WGRAD_STREAM=$f timeout 600 python bench.py --config 1b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/wgs_1b_${f}.log 2>&1
  CB_WGRAD_STREAM=$f timeout 600 python bench.py --config moe --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/wgs_moe_${f}.log 2>&1
done
