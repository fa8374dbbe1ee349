# Bench suite on one box: every BASELINE config the box's GPU count allows (used for the
# profiles/ evidence; each line is bench.py's JSON).  usage: bash scripts/suite.sh NGPUS TAG
N=${1:-1}; TAG=${2:-suite}
run() {  # config gpus extra...
  local c=$1 g=$2; shift 2
  if [ "$g" = 1 ]; then
    timeout 900 python bench.py --config $c --no-cpu-baseline "$@" > gpurun_out/${TAG}_${c}_${g}gpu.log 2>&1
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 \
      --master-port 29511 bench.py --gpus $g --config $c --no-cpu-baseline "$@" > gpurun_out/${TAG}_${c}_${g}gpu.log 2>&1
  fi
  echo "$c x$g: $(tail -1 gpurun_out/${TAG}_${c}_${g}gpu.log | cut -c1-220)"
}
for g in 1 2 4; do
  [ $g -gt $N ] && break
  run 1b $g
done
run 7b $N
run moe $N
run 70b_layer $N
