#!/bin/bash
# build an A/B variant of the library: tools/build_variant.sh <name> <extra nvcc flags...>
name=$1; shift
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr -I include "$@" -o paper_2604_09993_b200/_lib/libcito_b200_$name.so \
  paper_2604_09993_b200/csrc/cito_capi.cu -lcudart
