#!/bin/bash
# build an experimental variant of libpagedattn.so: scripts/build_variant.sh NAME "-DFLAG=.."
# -> paper_2309_06180_b200/libpagedattn_NAME.so, loaded with PA_LIB_VARIANT=NAME
set -e
NAME=$1; FLAGS=$2
D=/tmp/pa_variant_$NAME; mkdir -p $D; rm -f $D/*.o
SRC=paper_2309_06180_b200/csrc
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $FLAGS"
for f in $SRC/*.cu $SRC/*.cpp; do
  b=$(basename $f); $NV -c $f -o $D/${b%.*}.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2309_06180_b200/libpagedattn_$NAME.so $D/*.o
