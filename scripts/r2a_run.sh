set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2a_gpu_tests.log
timeout 300 python bench.py --config 7b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_7b.log 2>&1
timeout 300 python bench.py --config 1b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_1b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dkdv_k|dq_k|fwd_tc_k" -c 6 -o gpurun_out/r2a_attn_1b python scripts/attn_prof.py 1b > gpurun_out/r2a_ncu1b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dkdv_k|dq_k" -c 4 -o gpurun_out/r2a_attn_7b python scripts/attn_prof.py 7b > gpurun_out/r2a_ncu7b.log 2>&1
timeout 300 python scripts/attn_bench.py > gpurun_out/r2a_attn_bench.log 2>&1
ls gpurun_out
