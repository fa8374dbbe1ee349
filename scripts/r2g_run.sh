cd $GRAFT_REPO_ROOT
for mode in "--precision f32 --config txf_rope --seq 8" "--precision f32 --config mid --seq 128" "--precision bf16 --config mid --seq 128" "--precision f32 --config txf_moe --seq 8"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29531 scripts/fsdp_check.py $mode --steps 3 --mode step --collectives both > gpurun_out/tmp.log 2>&1
  echo "rc=$? $mode" >> gpurun_out/r2g_fsdp2.log; grep '^{' gpurun_out/tmp.log >> gpurun_out/r2g_fsdp2.log || tail -30 gpurun_out/tmp.log >> gpurun_out/r2g_fsdp2.log
done
timeout 600 python bench.py --config moe --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_bench_moe.log 2>&1
timeout 600 python bench.py --config moe --steps 5 --warmup 3 --no-cpu-baseline --moe-routing balanced > gpurun_out/r2g_bench_moe_bal.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 bench.py --gpus 2 --config 7b --steps 10 --warmup 3 > gpurun_out/r2g_bench_7b_2gpu.log 2>&1
timeout 600 python bench.py --config 7b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_bench_7b_1gpu.log 2>&1
