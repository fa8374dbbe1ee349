cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -rf -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/r2n_gpu_tests.log
