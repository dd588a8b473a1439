#!/bin/bash
# Build an A/B variant of libwave25.so with extra -D flags, in-tree:
#   bash scripts/build_variant.sh scalar -DW25_PACKED=0   -> paper_2009_04619_b200/libwave25_scalar.so
# then run with WAVE25_LIB=libwave25_scalar.so (measurement only).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC,-fvisibility=hidden -shared -prec-div=true -prec-sqrt=true -ftz=false "$@" \
  -o paper_2009_04619_b200/libwave25_${name}.so paper_2009_04619_b200/csrc/wave.cu
