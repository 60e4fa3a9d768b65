timeout 900 python -m pytest tests -m gpu -x -q -rs -k "fullsize_pins" > gpurun_out/pcgpin.log 2>&1; echo "exit $?" >> gpurun_out/pcgpin.log
