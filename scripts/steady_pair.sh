#!/usr/bin/env bash
# attention backward under power-capped steady clocks: single-CTA vs pair dK/dV sweep (dQ on pairs)
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for rep in a b; do
  for f in 0 1; do
    CB_ATTN_DKDV_PAIR=$f timeout 300 python scripts/attn_steady.py 7b 100 > gpurun_out/sp_7b_${f}_${rep}.log 2>&1
    CB_ATTN_DKDV_PAIR=$f timeout 300 python scripts/attn_steady.py 1b 60 > gpurun_out/sp_1b_${f}_${rep}.log 2>&1
  done
done
