#!/bin/bash
# Dev only: build a variant libfdpp.so with extra -D flags on the attention TUs
# (tools/ab_variant.sh OUTDIR -DFLAG ...); select it with FDPP_LIB=OUTDIR/libfdpp.so.
set -e -o pipefail
cd "$(dirname "$0")/.."
OUT=$1; shift
mkdir -p $OUT
B=paper_2311_01282_b200/csrc/build
pids=()
for f in paper_2311_01282_b200/csrc/attention_*.cu; do
  n=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr "$@" -Iinclude -c $f -o $OUT/$n.o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libfdpp.so \
  $OUT/attention_*.o $(ls $B/*.o | grep -v "/attention_") -lcuda
echo built $OUT/libfdpp.so
