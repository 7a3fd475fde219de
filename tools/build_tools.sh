#!/bin/bash
# Builds the standalone microbenchmarks in tools/ against the engine objects.
set -e
cd "$(dirname "$0")/.."
make -C paper_2501_12151_b200/csrc -j8 >/dev/null
OBJS=$(ls paper_2501_12151_b200/csrc/build/*.o)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2501_12151_b200/csrc \
  tools/gemm_shapes.cu $OBJS -o tools/gemm_shapes
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2501_12151_b200/csrc \
  tools/gemm_bench.cu $OBJS -o tools/gemm_bench
