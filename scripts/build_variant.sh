#!/bin/bash
# Build an A/B variant of libpatchdb.so.0 with one kernel file recompiled under
# extra nvcc flags: scripts/build_variant.sh NAME FILE.cu "FLAGS" -> paper_2306_10025_b200/lib/ab/NAME/libpatchdb.so.0
set -e
cd "$(dirname "$0")/../paper_2306_10025_b200/csrc"
name=$1; file=$2; flags=$3
make -s -j16 >/dev/null
out=../lib/ab/$name; mkdir -p $out obj/ab
base=$(basename $file .cu)
fm=""; case $base in lu|criterion) fm="--fmad=false";; esac
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr $fm $flags -c kernels/$file -o obj/ab/k_${base}_$name.o
objs=$(ls obj/[khc]_*.o | grep -v "obj/k_${base}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libpatchdb.so.0 $objs obj/ab/k_${base}_$name.o -lnccl \
  -Xlinker -soname=libpatchdb.so.0 -Xlinker --version-script=exports.map -cudart static -lpthread -ldl -lrt
echo $out/libpatchdb.so.0
