timeout 1200 python -m pytest tests -m gpu -x -q -k "entrywise_kmeans_matches_reference or front_order or relax or apply" > gpurun_out/pins.log 2>&1; echo "exit $?" >> gpurun_out/pins.log
