#!/usr/bin/env bash
# weight-gradient overwrite + inline AdamW: exactness tests, FSDP tests (2 GPUs), the 7B step on
# 1 and 2 GPUs with the overwrite on and off.   gpurun --gpus 2 -- 'bash scripts/ow_check.sh'
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_step_gpu.py tests/test_fsdp.py -q -rf -k "adamw or grad_ring or wgrad or checkpoint or fsdp or full_size_step or two_steps or functional" > gpurun_out/ow_tests.log 2>&1
for rep in a b; do
  for f in 1 0; do
    CB_WGRAD_OVERWRITE=$f timeout 600 python bench.py --config 7b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ow_7b_${f}_${rep}.log 2>&1
  done
done
for f in 1 0; do
  CB_WGRAD_OVERWRITE=$f timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
    --master-port=2958$f bench.py --gpus 2 --config 7b --steps 10 --warmup 3 > gpurun_out/ow_7b2_${f}.log 2>&1
done
