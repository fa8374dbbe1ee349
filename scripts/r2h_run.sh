cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for mode in "--precision bf16 --config mid --seq 128" "--precision f32 --config mid --seq 128"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29531 scripts/fsdp_check.py $mode --steps 3 --mode step --collectives both > gpurun_out/tmp.log 2>&1
  echo "rc=$? $mode" >> gpurun_out/r2h_fsdp2.log; grep '^{' gpurun_out/tmp.log >> gpurun_out/r2h_fsdp2.log || tail -30 gpurun_out/tmp.log >> gpurun_out/r2h_fsdp2.log
done
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 bench.py --gpus 2 --config 7b --steps 10 --warmup 3 > gpurun_out/r2h_7b_2gpu_$1.log 2>&1; }
CB_FSDP_RESHARD=1 CB_FSDP_GRAD_RING=1 run rs1_gr1
CB_FSDP_RESHARD=0 CB_FSDP_GRAD_RING=1 run rs0_gr1
CB_FSDP_RESHARD=0 CB_FSDP_GRAD_RING=0 run rs0_gr0
CB_FSDP_RESHARD=1 CB_FSDP_GRAD_RING=1 run rs1_gr1_b
timeout 600 python bench.py --config moe --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2h_bench_moe.log 2>&1
