#!/usr/bin/env bash
# FSDP forward gathers without the per-layer barrier after a synced step(): parity + A/B
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_fsdp.py -m gpu -q -rf > gpurun_out/fb_fsdp_tests.log 2>&1
for mode in "--precision f32 --config mid --seq 128" "--precision bf16 --config mid --seq 128" \
            "--precision f32 --config mid_moe --seq 128"; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=29661 scripts/fsdp_check.py $mode --steps 4 --mode step --collectives both \
    >> gpurun_out/fb_fsdp_parity.log 2>&1
done
for rep in a b; do
  for f in 0 1; do
    for n in 2 4; do
      CB_FSDP_FWD_BARRIER=$f timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n \
        --master-addr=127.0.0.1 --master-port=2967$n bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/fb_7b_${n}_${f}_${rep}.log 2>&1
    done
  done
done
