# A/B of the weight-gradient side stream (CB_WGRAD_STREAM=0|1), interleaved on one box.
# usage: bash scripts/wgrad_ab.sh TAG CONFIG ROUNDS [NGPUS]
TAG=${1:-wgab}; C=${2:-1b}; R=${3:-2}; N=${4:-1}
for i in $(seq 1 $R); do
  for w in ${WG_LIST:-0 1}; do
    f=gpurun_out/${TAG}_${C}_${N}gpu_wg${w}_$i.log
    if [ "$N" = 1 ]; then
      CB_WGRAD_STREAM=$w timeout 900 python bench.py --config $C --no-cpu-baseline > $f 2>&1
    else
      CB_WGRAD_STREAM=$w timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
        --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --config $C --no-cpu-baseline > $f 2>&1
    fi
    echo "$C x$N wgrad_stream=$w run $i: $(tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]), "tok/s", round(d["ms_per_step"],2), "ms", d["clocks"]["sm_mhz"], "MHz")' 2>&1 | tail -1)"
  done
done
