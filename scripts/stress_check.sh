#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -rf -x -k "dq_pair or attention" > gpurun_out/st_tests.log 2>&1
timeout 400 python scripts/attn_stress.py 3000 0 > gpurun_out/st_dq.log 2>&1; echo "rc=$?" >> gpurun_out/st_dq.log
timeout 400 python scripts/attn_stress.py 3000 1 > gpurun_out/st_both.log 2>&1; echo "rc=$?" >> gpurun_out/st_both.log
