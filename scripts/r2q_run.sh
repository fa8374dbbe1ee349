cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
CB_FSDP_MEMOP_BARRIER=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29571 scripts/fsdp_check.py --precision f32 --config mid --seq 128 --steps 3 --mode step --collectives ce > gpurun_out/r2q_memop_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/r2q_memop_parity.log
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29573 bench.py --gpus 2 --config 7b --steps 15 --warmup 3 > gpurun_out/r2q_7b_2gpu_$1.log 2>&1; }
if grep -q '"ok": true' gpurun_out/r2q_memop_parity.log; then
  CB_FSDP_MEMOP_BARRIER=0 run mb0_a
  CB_FSDP_MEMOP_BARRIER=1 run mb1_a
  CB_FSDP_MEMOP_BARRIER=0 run mb0_b
  CB_FSDP_MEMOP_BARRIER=1 run mb1_b
fi
