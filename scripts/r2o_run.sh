cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -k "f32" -rf 2>&1 | tail -15 > gpurun_out/r2o_f32.log
timeout 1500 python -m pytest tests/test_step_gpu.py -q -rf -k "f32 or registry or tiny or two_steps or functional or forward_loss or gqa or activation or remat" 2>&1 | tail -25 >> gpurun_out/r2o_f32.log
timeout 600 python scripts/parity_report.py mid64_f32 mid128_f32 moe_f32_t256 linear_f32 sigmoid_f32 > gpurun_out/r2o_parity_report.jsonl 2> gpurun_out/r2o_parity_report.err
