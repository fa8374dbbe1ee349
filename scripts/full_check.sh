#!/usr/bin/env bash
# Full GPU test suite + smoke + the default bench line and the reference arm (round-end rehearsal).
#   gpurun --gpus 2 -- 'bash scripts/full_check.sh'
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --durations=15 > gpurun_out/full_gpu_tests.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/full_smoke.log
timeout 900 python bench.py > gpurun_out/full_bench_default.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/full_bench_reference.log 2>&1
