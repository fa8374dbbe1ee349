#!/usr/bin/env bash
# dK/dV pair sweep x weight-gradient side stream (7B step), interleaved
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for rep in a b; do
  for cfg in "4 0" "4 1" "0 0" "0 1"; do
    set -- $cfg
    CB_WGRAD_STREAM=$1 CB_ATTN_DKDV_PAIR=$2 timeout 600 python bench.py --config 7b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/dkw_${1}_${2}_${rep}.log 2>&1
  done
done
