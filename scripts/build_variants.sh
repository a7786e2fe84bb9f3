#!/bin/bash
# Diagnostics builds of the library with experiment macros (not product code paths):
#   bash scripts/build_variants.sh NAME "-DMACRO ..."   → tests/probe/libentmax_NAME.so
set -e
NAME=$1; shift
S=paper_2502_12082_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -I$S \
  --expt-relaxed-constexpr "$@" -shared -o tests/probe/libentmax_$NAME.so \
  $S/entmax_attn.cu $S/simt.cu $S/sm100.cu $S/rowwise.cu
