# round-2 GPU check: full -m gpu suite on one GPU + smoke
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -40 > gpurun_out/r2b_gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2b_smoke.log 2>&1
