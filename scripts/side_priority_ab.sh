# side-stream priority A/B (optimizer stream at 1 GPU, NCCL + optimizer stream at 2 GPUs)
for c in moe 1b; do for p in 0 -1 0 -1; do
  CB_SIDE_STREAM_PRIORITY=$p timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/pr.log 2>&1
  echo "$c priority $p: $(tail -1 gpurun_out/pr.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],2))")"
done; done
for p in 0 -1; do
  CB_SIDE_STREAM_PRIORITY=$p timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/pr2.log 2>&1
  echo "1b x2 priority $p: $(tail -1 gpurun_out/pr2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],2))")"
done
