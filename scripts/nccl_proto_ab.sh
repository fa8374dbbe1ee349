# NCCL protocol A/B of the 4-GPU 1B step: the default picks RING_LL kernels for the per-layer
# bucket all-gather / reduce-scatter (see scripts/gap_profile.py under torchrun)
run() {
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/nccl_proto.log 2>&1
  echo "$*: $(tail -1 gpurun_out/nccl_proto.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],1))")"
}
run X=1
run NCCL_PROTO=Simple
run NCCL_PROTO=Simple NCCL_ALGO=NVLS
run X=1
run NCCL_PROTO=Simple
