#!/usr/bin/env bash
# the default 7B step at 1, 2 and 4 GPUs (weak scaling) at HEAD.  gpurun --gpus 4 -- 'bash scripts/scale7b.sh'
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s7_1gpu.log 2>&1
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=2961$n bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/s7_${n}gpu.log 2>&1
done
nvidia-smi --query-gpu=index,clocks.sm,power.draw,power.limit,temperature.gpu --format=csv > gpurun_out/s7_smi.txt 2>&1
