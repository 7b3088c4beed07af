#!/bin/bash
# build an experimental variant of libpagedattn.so: scripts/build_variant.sh NAME "-DFLAG=.."
set -e
NAME=$1; FLAGS=$2
D=/tmp/pa_variant_$NAME; mkdir -p $D
SRC=paper_2309_06180_b200/csrc
for f in pa_attention pa_prefill pa_cache; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $FLAGS -c $SRC/$f.cu -o $D/$f.o
done
for f in pa_api pa_alloc; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $FLAGS -c $SRC/$f.cpp -o $D/$f.o
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2309_06180_b200/libpagedattn_$NAME.so $D/*.o
