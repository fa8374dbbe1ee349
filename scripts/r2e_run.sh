cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/r2e_gpus.txt
timeout 2400 python -m pytest tests -m gpu -q -rf -p no:cacheprovider 2>&1 | tail -60 > gpurun_out/r2e_gpu_tests.log
