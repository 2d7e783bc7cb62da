#!/bin/bash
# Build A/B variants of the library into scratch_so/ (git-ignored, travels with
# gpurun):  bash tools/variants.sh NAME "-DFLAG ..." [NAME "-D..."] ...
mkdir -p scratch_so
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
    -Xcompiler -fPIC -shared $flags -o scratch_so/$name.so paper_1512_01641_b200/csrc/abi.cu \
    paper_1512_01641_b200/csrc/host_text.cpp || exit 1
  echo "built scratch_so/$name.so ($flags)"
done
