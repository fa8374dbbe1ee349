# 4-GPU FSDP parity against the oracle: TrainEngine.step() for 3 chained steps, f32 and bf16,
# two configs, copy-engine and NCCL collectives (scripts/fsdp_check.py --mode step)
for prec in f32 bf16; do for cfg in txf_rope mid; do
  seq=$([ $cfg = mid ] && echo 128 || echo 8)
  timeout 600 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 \
    scripts/fsdp_check.py --precision $prec --config $cfg --seq $seq --steps 3 --mode step --collectives both 2>&1 \
    | grep -v -i -E "warn|OMP|\*\*\*\*" | tail -1
done; done
