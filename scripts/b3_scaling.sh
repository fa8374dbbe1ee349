#!/usr/bin/env bash
# 7B step at the default 3 sequences per GPU on 1, 2 and 4 GPUs (weak scaling, memory per GPU),
# then the default bench line and the reference arm.   gpurun --gpus 4 -- 'bash scripts/b3_scaling.sh'
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python bench.py --config 7b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b3_7b_1gpu.log 2>&1
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=2957$n bench.py --gpus $n --config 7b --steps 10 --warmup 3 > gpurun_out/b3_7b_${n}gpu.log 2>&1
done
timeout 900 python bench.py > gpurun_out/b3_bench_default.log 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/b3_bench_reference.log 2>&1
