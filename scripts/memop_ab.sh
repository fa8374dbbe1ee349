# FSDP barrier A/B at 4 GPUs (torch symm-mem barrier kernel vs stream memory operations)
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
run() { CB_FSDP_MEMOP_BARRIER=$2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 \
  --master-addr=127.0.0.1 --master-port=29581 bench.py --gpus 4 --config $1 --steps 10 --warmup 3 > gpurun_out/memop4_$1_$2_$3.log 2>&1; }
for rep in a b; do for cfg in 70b_layer moe; do for mb in 0 1; do run $cfg $mb $rep; done; done; done
