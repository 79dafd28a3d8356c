#!/bin/bash
# build experimental variants of the library (same sources, different macros)
cd "$(dirname "$0")/.."
mkdir -p paper_2408_12179_b200/variants
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -shared -diag-suppress 177 -Xcompiler -Wno-deprecated-declarations -ldl"
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  $NV $flags -o paper_2408_12179_b200/variants/libhprlp_b200_$name.so paper_2408_12179_b200/csrc/hpr_capi.cu paper_2408_12179_b200/csrc/hpr_mps.cpp &
done
wait
