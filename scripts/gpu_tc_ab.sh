#!/bin/bash
# A/B of compile-time variants of the tcgen05 N1 decode: default build vs each NVXFLAGS argument
mkdir -p gpurun_out
rm -f gpurun_out/tc_ab.jsonl
for v in "" "$@"; do
  make clean > /dev/null && make -j8 NVXFLAGS="$v" > gpurun_out/build_ab.txt 2>&1
  for c in "c5_beam --grouped 4" "c3_fork --grouped 6"; do
    echo "{\"variant\": \"$v\"}" >> gpurun_out/tc_ab.jsonl
    PA_TC_SPLIT=0 timeout 150 python bench.py --config $c --no-cpu-baseline --no-prefill --no-e2e --steps 300 >> gpurun_out/tc_ab.jsonl 2>> gpurun_out/tc_ab.err
  done
done
make clean > /dev/null && make -j8 > gpurun_out/build.txt 2>&1
