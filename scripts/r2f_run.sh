cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -k "grouped or dispatch_padded" -rf 2>&1 | tail -30 > gpurun_out/r2f_grouped.log
timeout 1200 python -m pytest tests/test_step_gpu.py -q -k "moe or forward_loss or functional or full_size or fast_path or activation or registry" -rf 2>&1 | tail -30 > gpurun_out/r2f_step.log
for mode in "--precision f32 --config txf_rope --seq 8" "--precision f32 --config mid --seq 128" "--precision bf16 --config mid --seq 128"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29531 scripts/fsdp_check.py $mode --steps 3 --mode step --collectives both >> gpurun_out/r2f_fsdp2.log 2>&1
  echo "rc=$?" >> gpurun_out/r2f_fsdp2.log
done
timeout 600 python bench.py --config moe --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench_moe.log 2>&1
timeout 600 python bench.py --config moe --steps 5 --warmup 3 --no-cpu-baseline --moe-routing balanced > gpurun_out/r2f_bench_moe_bal.log 2>&1
