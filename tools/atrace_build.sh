#!/bin/bash
# Trace-instrumented libfdpp for tools/attn_trace.py (dev only).
set -e -o pipefail
cd "$(dirname "$0")/.."
mkdir -p tools/atrace
# the f16 async attention TU carries the trace buffer; the others are the normal objects
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -DFDPP_ATRACE -Iinclude -c paper_2311_01282_b200/csrc/attention_f16_async.cu \
  -o tools/atrace/attention_f16_async.o
B=paper_2311_01282_b200/csrc/build
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/atrace/libfdpp.so \
  tools/atrace/attention_f16_async.o $(ls $B/*.o | grep -v attention_f16_async) -lcuda
echo built tools/atrace/libfdpp.so
