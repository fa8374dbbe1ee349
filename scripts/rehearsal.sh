#!/usr/bin/env bash
# the round-end driver commands on one GPU, at HEAD
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -x -q -m gpu > gpurun_out/rh_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rh_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rh_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/rh_smoke.log
timeout 900 python bench.py > gpurun_out/rh_bench.log 2>&1; echo "rc=$?" >> gpurun_out/rh_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/rh_reference.log 2>&1; echo "rc=$?" >> gpurun_out/rh_reference.log
