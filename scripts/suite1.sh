# single-GPU bench lines of every BASELINE config (profiles/ evidence)
TAG=${1:-suite1}
for c in 1b 7b moe 70b_layer; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_${c}_1gpu.log 2>&1
  echo "$c: $(tail -1 gpurun_out/${TAG}_${c}_1gpu.log | cut -c1-160)"
done
