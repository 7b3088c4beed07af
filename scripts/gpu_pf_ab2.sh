#!/bin/bash
# compile-time A/B of the prompt kernels on the long-prompt workloads
mkdir -p gpurun_out
rm -f gpurun_out/pf_ab2.jsonl
for v in "" "$@"; do
  make clean > /dev/null && make -j8 NVXFLAGS="$v" > gpurun_out/build_ab.txt 2>&1
  echo "{\"variant\": \"$v\"}" >> gpurun_out/pf_ab2.jsonl
  timeout 300 python scripts/prefill_bench.py --no-cpu-baseline --configs p_2k,p_chunk256,p_prefix5 >> gpurun_out/pf_ab2.jsonl 2>> gpurun_out/pf_ab2.err
done
make clean > /dev/null && make -j8 > gpurun_out/build.txt 2>&1
