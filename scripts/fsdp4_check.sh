# 4-GPU FSDP parity against the oracle (f32 and bf16, two configs, two chained steps)
for prec in f32 bf16; do for cfg in txf_rope mid; do
  timeout 600 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 scripts/fsdp_check.py --precision $prec --config $cfg --steps 2 --decomposed 2>&1 | grep -v -i -E "warn|OMP|\*\*\*\*" | tail -1
done; done
