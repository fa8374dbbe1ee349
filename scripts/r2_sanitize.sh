# compute-sanitizer on tiny shapes (each tool bounded by timeout); logs to gpurun_out/
cd $GRAFT_REPO_ROOT
python scripts/sanitize_small.py > gpurun_out/san_plain.log 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_small.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_summary.txt
done
