#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 120 scripts/bin/attn_bwd_trace pair > gpurun_out/rx_trace.txt 2>&1
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -rf -x -k "attention" > gpurun_out/rx_tests.log 2>&1
timeout 300 python scripts/attn_steady.py 7b 100 > gpurun_out/rx_steady_7b.log 2>&1
timeout 300 python scripts/attn_steady.py 1b 60 > gpurun_out/rx_steady_1b.log 2>&1
