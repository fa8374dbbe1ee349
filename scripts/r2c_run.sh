cd $GRAFT_REPO_ROOT
timeout 900 python scripts/parity_report.py > gpurun_out/r2c_parity_report.jsonl 2> gpurun_out/r2c_parity_report.err
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "linear_with_bias or attention_fwd_bwd" 2>&1 | tail -40 > gpurun_out/r2c_kern.log
timeout 1200 python -m pytest tests/test_step_gpu.py -q -k "remat or gqa" 2>&1 | tail -40 > gpurun_out/r2c_remat.log
