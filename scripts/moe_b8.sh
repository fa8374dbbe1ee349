#!/usr/bin/env bash
# MoE step at 4 and 8 sequences per GPU, router and balanced routing
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for b in 4 8; do
  for r in router balanced; do
    timeout 600 python bench.py --config moe --batch $b --moe-routing $r --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/moeb_${b}_${r}.log 2>&1
  done
done
