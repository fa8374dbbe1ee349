cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/r2i_gpu_tests.log
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 bench.py --gpus 2 --config $1 --steps 10 --warmup 3 > gpurun_out/r2i_$1_2gpu.log 2>&1; }
run 7b
run 1b
timeout 600 python bench.py --config 70b_layer --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_70b_1gpu.log 2>&1
timeout 600 python bench.py --config 70b_layer --steps 5 --warmup 3 --no-cpu-baseline --remat save_all > gpurun_out/r2i_70b_1gpu_saveall.log 2>&1
timeout 300 python scripts/attn_steady.py 7b 60 > gpurun_out/r2i_attn_steady.log 2>&1
timeout 300 python scripts/attn_steady.py 1b 30 >> gpurun_out/r2i_attn_steady.log 2>&1
