CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 2400 $CS --tool $tool --error-exitcode 9 --print-limit 50 python scripts/sanitize_small.py > gpurun_out/san_$tool.log 2>&1; echo "exit $?" >> gpurun_out/san_$tool.log
done
