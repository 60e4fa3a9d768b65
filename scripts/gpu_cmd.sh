timeout 300 python scripts/fp64_probe.py > gpurun_out/fp64.log 2>&1; echo "exit $?" >> gpurun_out/fp64.log
cp profiles/fp64_peaks.json gpurun_out/fp64_peaks.json
