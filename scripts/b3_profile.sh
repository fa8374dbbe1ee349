#!/usr/bin/env bash
# ncu evidence for the 3-sequence 7B default: launch list of exactly one step and a full capture
# of the QKV GEMM at M = 12288.   gpurun -- 'bash scripts/b3_profile.sh'
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/b3_launches_7b.csv python scripts/step_once.py --config 7b --batch 3 > gpurun_out/b3_step_once.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 1 -c 1 \
  -o gpurun_out/b3_gemm_qkv7b3 python scripts/gemm_one.py qkv7b3 > gpurun_out/b3_gemm_one.log 2>&1
# per-kernel breakdown (top_ms) of the MoE and 1B steps
timeout 600 python bench.py --config moe --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b3_moe_1gpu.log 2>&1
timeout 600 python bench.py --config 1b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b3_1b_1gpu.log 2>&1
