cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "adamw" 2>&1 | tail -3 > gpurun_out/r2j_adamw_test.log
timeout 900 python bench.py > gpurun_out/r2j_bench_default.log 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2j_bench_reference.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2j_launches_7b.csv python scripts/step_once.py --config 7b > gpurun_out/r2j_launches_7b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 1 -c 1 -o gpurun_out/r2j_gemm_qkv7b python scripts/gemm_one.py qkv7b > gpurun_out/r2j_ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 1 -c 1 -o gpurun_out/r2j_gemm_down7b python scripts/gemm_one.py down7b >> gpurun_out/r2j_ncu_gemm.log 2>&1
