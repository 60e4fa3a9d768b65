timeout 900 python -m pytest tests -x -q -m gpu -k "gmres or pcg or krylov" > gpurun_out/t_kry.log 2>&1; echo "exit $?" >> gpurun_out/t_kry.log
timeout 600 python scripts/pcg_c2.py 2 entrywise > gpurun_out/pcg2.log 2>&1; echo "exit $?" >> gpurun_out/pcg2.log
