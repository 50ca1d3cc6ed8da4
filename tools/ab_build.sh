#!/bin/bash
# Build the current csrc/ into an alternative library path for A/B timing on the GPU box:
#   tools/ab_build.sh build/ab/libX.so [extra nvcc flags]   then   DOCKSCREEN_LIB=build/ab/libX.so python bench.py ...
set -e
OUT=$(realpath -m "$1"); shift
cd "$(dirname "$0")/../paper_2209_05069_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -prec-div=true -prec-sqrt=true -std=c++17 \
  -Xcompiler -fPIC,-fopenmp,-O3,-ffp-contract=off "$@" -shared -o "$OUT" \
  ds_align.cu ds_optimize.cu ds_latency.cu ds_ops.cu ds_generate.cu ds_api.cu ds_host.cpp -lgomp
