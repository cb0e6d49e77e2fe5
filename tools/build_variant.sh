#!/bin/bash
# Build the library with extra nvcc flags into another file, for A/B runs
# (tools/ab_libs.sh loads it via BC_LIBRARY).  usage: build_variant.sh OUT.so -DFOO ...
set -e
cd "$(dirname "$0")/.."
OUT=$1; shift
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a \
  -Xcompiler -fPIC,-O2,-ffp-contract=off,-fvisibility=hidden --expt-relaxed-constexpr -shared \
  -I include "$@" -o "$OUT" paper_2501_18977_b200/csrc/*.cu
