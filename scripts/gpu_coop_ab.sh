#!/bin/bash
# A/B of compile-time variants of the coop decode kernel on C2: default build vs each NVXFLAGS argument
mkdir -p gpurun_out
rm -f gpurun_out/coop_ab.jsonl
for v in "" "$@"; do
  make clean > /dev/null && make -j8 NVXFLAGS="$v" > gpurun_out/build_ab.txt 2>&1
  for c in c2_alpaca c2_sharegpt; do
    echo "{\"variant\": \"$v\"}" >> gpurun_out/coop_ab.jsonl
    timeout 150 python bench.py --config $c --no-cpu-baseline --no-prefill --no-e2e --steps 500 >> gpurun_out/coop_ab.jsonl 2>> gpurun_out/coop_ab.err
  done
done
make clean > /dev/null && make -j8 > gpurun_out/build.txt 2>&1
