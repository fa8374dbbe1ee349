cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
nvidia-smi -L > gpurun_out/r2k_gpus.txt
timeout 900 python -m pytest tests/test_step_gpu.py tests/test_gemm_gpu.py -q -k "moe or grouped or dispatch" -rf 2>&1 | tail -5 > gpurun_out/r2k_moe_tests.log
timeout 1500 python -m pytest tests/test_fsdp.py -m gpu -q -rf 2>&1 | tail -12 > gpurun_out/r2k_fsdp_tests.log
for mode in "--precision f32 --config mid --seq 128" "--precision bf16 --config mid --seq 128" "--precision f32 --config mid_moe --seq 128"; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29541 scripts/fsdp_check.py $mode --steps 3 --mode step --collectives both > gpurun_out/tmp.log 2>&1
  echo "rc=$? $mode" >> gpurun_out/r2k_fsdp4.jsonl; grep '^{' gpurun_out/tmp.log >> gpurun_out/r2k_fsdp4.jsonl || tail -30 gpurun_out/tmp.log >> gpurun_out/r2k_fsdp4.jsonl
done
for cfg in 7b 1b moe 70b_layer; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2k_${cfg}_1gpu.log 2>&1
  for n in 2 4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=2955$n bench.py --gpus $n --config $cfg --steps 10 --warmup 3 > gpurun_out/r2k_${cfg}_${n}gpu.log 2>&1
  done
done
