#!/usr/bin/env bash
# The round-2 final measurement suite (HEAD) (run on a GPU box from the repo root; outputs in gpurun_out/).
#   gpurun --gpus 4 -- 'bash scripts/final_suite.sh'
# Each step is bounded by `timeout`; see profiles/README.md for what each produced.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
# 1. parity: the GPU test suite (multi-GPU tests run when >= 2 / 4 GPUs are visible)
timeout 2400 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/final_gpu_tests.log 2>&1
# 2. FSDP step parity at N GPUs (both collective implementations)
if [ "$NG" -ge 2 ]; then
  for mode in "--precision f32 --config mid --seq 128" "--precision bf16 --config mid --seq 128" \
              "--precision f32 --config mid_moe --seq 128"; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 \
      --master-port=29541 scripts/fsdp_check.py $mode --steps 3 --mode step --collectives both \
      >> gpurun_out/final_fsdp_parity.log 2>&1
  done
fi
# 3. weak scaling of every bench config at 1 .. NG GPUs
for cfg in 7b 1b moe 70b_layer; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final_${cfg}_1gpu.log 2>&1
  for n in 2 4; do
    [ "$n" -le "$NG" ] || continue
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
      --master-port=2955$n bench.py --gpus $n --config $cfg --steps 10 --warmup 3 > gpurun_out/final_${cfg}_${n}gpu.log 2>&1
  done
done
# 4. the default bench line, the reference arm, a one-step launch list and the ncu captures
timeout 900 python bench.py > gpurun_out/final_bench_default.log 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final_bench_reference.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/final_launches_7b.csv python scripts/step_once.py --config 7b --batch 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 1 -c 1 \
  -o gpurun_out/final_gemm_qkv7b3 python scripts/gemm_one.py qkv7b3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dkdv_k|dq_k" -c 2 \
  -o gpurun_out/final_attn_7b python scripts/attn_prof.py 7b > /dev/null 2>&1
