#!/usr/bin/env bash
# Last validation at HEAD (gpurun --gpus 4): every GPU test, FSDP step parity at 4 GPUs, smoke,
# the default bench line, the 7B step at 2 and 4 GPUs, the reference arm.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/f2_gpu_tests.log 2>&1
for mode in "--precision f32 --config mid --seq 128" "--precision bf16 --config mid --seq 128" \
            "--precision f32 --config mid_moe --seq 128"; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=29641 scripts/fsdp_check.py $mode --steps 3 --mode step --collectives both \
    >> gpurun_out/f2_fsdp_parity.log 2>&1
done
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f2_smoke.log
timeout 900 python bench.py > gpurun_out/f2_bench_default.log 2>&1
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=2965$n bench.py --gpus $n > gpurun_out/f2_7b_${n}gpu.log 2>&1
done
timeout 900 python bench.py --impl reference > gpurun_out/f2_bench_reference.log 2>&1
