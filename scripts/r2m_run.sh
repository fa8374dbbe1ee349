cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "dq_gemm" -rf 2>&1 | tail -30 > gpurun_out/r2m_dqgemm.log
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "attention" -rf 2>&1 | tail -15 >> gpurun_out/r2m_dqgemm.log
timeout 300 python scripts/attn_steady.py 7b 40 > gpurun_out/r2m_attn_steady.log 2>&1
timeout 300 python scripts/attn_steady.py 1b 20 >> gpurun_out/r2m_attn_steady.log 2>&1
CB_ATTN_DQ_GEMM=0 timeout 300 python scripts/attn_steady.py 7b 40 >> gpurun_out/r2m_attn_steady.log 2>&1
CB_ATTN_DQ_GEMM=0 timeout 300 python scripts/attn_steady.py 1b 20 >> gpurun_out/r2m_attn_steady.log 2>&1
