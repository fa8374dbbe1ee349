# GEMM raster group height A/B on the 7B step (CB_GEMM_RASTER; interleaved, default 16 twice)
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
for g in 16 8 32 4 16; do
  CB_GEMM_RASTER=$g timeout 600 python bench.py --config 7b --steps 15 --warmup 3 --no-cpu-baseline > gpurun_out/raster_7b_$g.log 2>&1
  CB_GEMM_RASTER=$g timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none \
    -k regex:gemm_tc2 -s 1 -c 1 --csv python scripts/gemm_one.py down7b > gpurun_out/raster_ncu_down_$g.csv 2>&1
done
