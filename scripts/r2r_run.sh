cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for g in 16 8 32 4 16; do
  CB_GEMM_RASTER=$g timeout 600 python bench.py --config 7b --steps 15 --warmup 3 --no-cpu-baseline > gpurun_out/r2r_7b_raster$g.log 2>&1
  CB_GEMM_RASTER=$g timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_tc2 -s 1 -c 1 --csv python scripts/gemm_one.py down7b > gpurun_out/r2r_ncu_down_raster$g.csv 2>&1
done
