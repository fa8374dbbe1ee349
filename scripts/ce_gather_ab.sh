# A/B of the FSDP parameter all-gather: NCCL (CB_FSDP_CE_GATHER=0) vs copy-engine peer reads of
# symmetric-memory working copies (=1), interleaved on one box.
# usage: bash scripts/ce_gather_ab.sh TAG CONFIG ROUNDS NGPUS   (AB_VAR=CB_FSDP_CE_REDUCE: the
# reduce-scatter variant instead)
TAG=${1:-ceab}; C=${2:-1b}; R=${3:-2}; N=${4:-2}; V=${AB_VAR:-CB_FSDP_CE_GATHER}
for i in $(seq 1 $R); do
  for ce in 0 1; do
    f=gpurun_out/${TAG}_${C}_${N}gpu_ce${ce}_$i.log
    env $V=$ce timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $N --config $C --no-cpu-baseline > $f 2>&1
    echo "$C x$N $V=$ce run $i: $(tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]), "tok/s", round(d["ms_per_step"],2), "ms", d["clocks"]["sm_mhz"], "MHz")' 2>&1 | tail -1)"
  done
done
