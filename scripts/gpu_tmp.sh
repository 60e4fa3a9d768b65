for i in 1 2; do
  CONFIGS="3 2" STEPS=300 scripts/sweep_ab.sh "TAG=default" >> gpurun_out/async.log 2>&1
  PDB_LIB_PATH=paper_2306_10025_b200/lib/ab/async/libpatchdb.so.0 CONFIGS="3 2" STEPS=300 scripts/sweep_ab.sh "TAG=async" >> gpurun_out/async.log 2>&1
done
PDB_LIB_PATH=paper_2306_10025_b200/lib/ab/async/libpatchdb.so.0 timeout 900 python -m pytest tests -m gpu -x -q -k "relax or apply or history or identity" >> gpurun_out/async.log 2>&1
