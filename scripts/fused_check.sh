#!/usr/bin/env bash
# AdamW fused into the weight-gradient GEMMs: exactness tests, then the 7B / 1B steps with the
# fusion on and off (interleaved).   gpurun -- 'bash scripts/fused_check.sh'
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py -q -rf -x -k "adamw or grad_ring or wgrad or checkpoint or full_size_step" > gpurun_out/fused_tests.log 2>&1
for rep in a b; do
  for f in 1 0; do
    CB_FUSED_ADAMW=$f timeout 600 python bench.py --config 7b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/fused_7b_${f}_${rep}.log 2>&1
  done
done
for f in 1 0; do
  CB_FUSED_ADAMW=$f timeout 600 python bench.py --config 1b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/fused_1b_${f}.log 2>&1
done
