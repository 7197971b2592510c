#!/bin/bash
# Build a trace-instrumented copy of libfdpp into tools/trace/ (dev only).
set -e -o pipefail
cd "$(dirname "$0")/.."
mkdir -p tools/trace
for f in gemm host; do
  src=paper_2311_01282_b200/csrc/$f.cu; [ -f $src ] || src=paper_2311_01282_b200/csrc/$f.cpp
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -DFDPP_TRACE -Iinclude -c $src -o tools/trace/$f.o &
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -Iinclude -c paper_2311_01282_b200/csrc/attention.cu -o tools/trace/attention.o &
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -Iinclude -c paper_2311_01282_b200/csrc/decode_ops.cu -o tools/trace/decode_ops.o &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/trace/libfdpp.so tools/trace/*.o
echo built tools/trace/libfdpp.so
