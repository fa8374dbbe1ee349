cd $GRAFT_REPO_ROOT
timeout 900 python scripts/parity_report.py mid64_f32 moe_f32_t256 linear_f32 sigmoid_bf16 swiglu_bf16 relu_d32_bf16 > gpurun_out/r2d_parity_report.jsonl 2> gpurun_out/r2d_parity_report.err
timeout 900 python -m pytest tests/test_kernels_gpu.py -q 2>&1 | tail -30 > gpurun_out/r2d_kern.log
bash scripts/r2_sanitize.sh
