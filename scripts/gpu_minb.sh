for v in default minb5 minb6 minb8 default; do
  if [ $v = default ]; then L=""; else L=paper_2306_10025_b200/lib/ab/$v/libpatchdb.so.0; fi
  PDB_LIB_PATH=$L TAG=$v REPS=2 python scripts/lib_ab.py >> gpurun_out/minb.log 2>&1
done
