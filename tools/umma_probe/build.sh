#!/bin/bash
# Builds the tcgen05 descriptor probe / MMA-rate micro-benchmark (tools only; the product
# library paper_2009_01462_b200/librespar_b200.so does not contain it).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(dirname "$(dirname "$HERE")")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
  -I"$ROOT/include" -I"$ROOT/paper_2009_01462_b200/csrc" --expt-relaxed-constexpr -shared \
  "$HERE/umma_probe.cu" -o "$HERE/librp_probe.so" -lcuda
echo "$HERE/librp_probe.so"
