#!/usr/bin/env bash
# MoE small-kernel work: kernel tests, the MoE parity tests, a launch list of one MoE step and
# the MoE bench line.   gpurun -- 'bash scripts/moe_check.sh'
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_gemm_gpu.py -q -rf -k "sort or router or moe or dispatch or embedding or combine" > gpurun_out/moe_tests.log 2>&1
timeout 900 python -m pytest tests/test_step_gpu.py -q -rf -k "moe" > gpurun_out/moe_step_tests.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/moe_launches.csv python scripts/step_once.py --config moe > /dev/null 2>&1
timeout 600 python bench.py --config moe --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/moe_bench.log 2>&1
