cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561 scripts/gap_profile.py --config 7b --steps 2 > gpurun_out/r2p_gap_7b_2gpu.log 2>&1
timeout 600 python scripts/gap_profile.py --config 7b --steps 2 > gpurun_out/r2p_gap_7b_1gpu.log 2>&1
