cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --durations=15 2>&1 | tail -60 > gpurun_out/r2l_gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2l_smoke.log 2>&1
