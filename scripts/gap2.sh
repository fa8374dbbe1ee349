#!/usr/bin/env bash
# 7B at 3 sequences on 2 GPUs: bench line + per-rank idle gaps.  gpurun --gpus 2 -- 'bash scripts/gap2.sh'
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29601 \
  bench.py --gpus 2 --config 7b --steps 10 --warmup 3 > gpurun_out/gap2_bench.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29602 \
  scripts/gap_profile.py --config 7b --batch 3 --steps 2 > gpurun_out/gap2_gaps.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,power.draw,temperature.gpu --format=csv > gpurun_out/gap2_smi.txt 2>&1
lscpu | head -20 > gpurun_out/gap2_cpu.txt 2>&1
