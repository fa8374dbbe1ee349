#!/usr/bin/env bash
# north-star-width oracle parity + the full-size property tests.  gpurun -- 'bash scripts/ns_check.sh'
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_step_gpu.py -q -rf -k "north_star or head_geometry or full_size" --durations=10 > gpurun_out/ns_tests.log 2>&1
