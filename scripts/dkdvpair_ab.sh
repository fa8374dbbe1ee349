#!/usr/bin/env bash
# attention backward dK/dV sweep single-CTA vs CTA pairs (dQ on pairs either way), full steps (interleaved)
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -rf -x -k "dq_pair or attention" > gpurun_out/dkvab_tests.log 2>&1
for rep in a b; do
  for f in 0 1; do
    CB_ATTN_DKDV_PAIR=$f timeout 600 python bench.py --config 7b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/dkvab_7b_${f}_${rep}.log 2>&1
  done
done
for f in 0 1; do
  CB_ATTN_DKDV_PAIR=$f timeout 600 python bench.py --config 1b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/dkvab_1b_${f}.log 2>&1
  CB_ATTN_DKDV_PAIR=$f timeout 600 python bench.py --config 70b_layer --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/dkvab_70b_${f}.log 2>&1
done
