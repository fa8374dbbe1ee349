#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -rf -x -k "dq_pair" > gpurun_out/dqp_tests.log 2>&1
timeout 300 python scripts/dq_pair_bench.py > gpurun_out/dqp_bench.log 2>&1
