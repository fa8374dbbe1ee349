#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for r in 1 2 3; do
  timeout 400 python bench.py --config 7b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s2_7b_$r.log 2>&1; echo "rc=$?" >> gpurun_out/s2_7b_$r.log
  CB_ATTN_DKDV_PAIR=1 timeout 400 python bench.py --config 7b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s2_7b_dkdv_$r.log 2>&1; echo "rc=$?" >> gpurun_out/s2_7b_dkdv_$r.log
done
timeout 500 python scripts/attn_stress.py 20000 1 > gpurun_out/s2_stress.log 2>&1; echo "rc=$?" >> gpurun_out/s2_stress.log
