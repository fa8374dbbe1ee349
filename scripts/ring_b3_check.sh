# one-GPU gradient ring: exactness test, then the 7B step at 2 and 3 sequences per GPU, and
# the default bench line + the reference arm with the current bench.py
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_step_gpu.py -q -rf -k "grad_ring or full_size or wgrad or checkpoint" > gpurun_out/ring_tests.log 2>&1
timeout 600 python bench.py --config 7b --batch 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ring_7b_b2.log 2>&1
timeout 600 python bench.py --config 7b --batch 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ring_7b_b3.log 2>&1
CB_GRAD_RING=0 timeout 600 python bench.py --config 7b --batch 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ring0_7b_b2.log 2>&1
timeout 900 python bench.py > gpurun_out/ring_bench_default.log 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ring_bench_reference.log 2>&1
timeout 1500 python -m pytest tests/test_fsdp.py -m gpu -q -rf > gpurun_out/ring_fsdp_tests.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29591 bench.py --gpus 2 --config 7b --steps 10 --warmup 3 > gpurun_out/ring_7b_2gpu.log 2>&1
