# NCCL channel-count A/B of the 4-GPU 1B step (fewer channels -> fewer SMs taken, but less bandwidth)
run() {
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/nccl_ab.log 2>&1
  echo "$*: $(tail -1 gpurun_out/nccl_ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],1))")"
}
NCCL_DEBUG=INFO timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --no-cpu-baseline --steps 3 > gpurun_out/nccl_info.log 2>&1
grep -i -E "nvls|channels|Using network|NCCL version" gpurun_out/nccl_info.log | sort | uniq -c | sort -rn | head -15
run X=1
run NCCL_MAX_NCHANNELS=4
run NCCL_MAX_NCHANNELS=2
run X=1
