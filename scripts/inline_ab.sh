#!/usr/bin/env bash
# one-GPU AdamW beside the backward (comm stream, default) vs inline on the compute stream
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for rep in a b; do
  for f in 0 1; do
    CB_ADAMW_INLINE=$f timeout 600 python bench.py --config 7b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/inline_7b_${f}_${rep}.log 2>&1
  done
done
for f in 0 1; do
  CB_ADAMW_INLINE=$f timeout 600 python bench.py --config 1b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/inline_1b_${f}.log 2>&1
  CB_ADAMW_INLINE=$f timeout 600 python bench.py --config moe --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/inline_moe_${f}.log 2>&1
done
