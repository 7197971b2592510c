#!/bin/bash
# Trace-instrumented libfdpp for tools/attn_trace.py (dev only).
set -e -o pipefail
cd "$(dirname "$0")/.."
mkdir -p tools/atrace
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -DFDPP_ATRACE -Iinclude -c paper_2311_01282_b200/csrc/attention.cu -o tools/atrace/attention.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/atrace/libfdpp.so \
  tools/atrace/attention.o paper_2311_01282_b200/csrc/build/gemm.cu.o paper_2311_01282_b200/csrc/build/decode_ops.cu.o \
  paper_2311_01282_b200/csrc/build/host.cpp.o -lcuda
echo built tools/atrace/libfdpp.so
