#!/bin/bash
# TMA producer-warp count A/B (4 / 6 / 8) for the prompt kernels v3 / v6
mkdir -p gpurun_out
rm -f gpurun_out/prod_ab2.jsonl
for n in 4 6 8; do
  make clean > /dev/null && make -j8 NVXFLAGS=-DPA_PF_PROD=$n > gpurun_out/build_prod$n.txt 2>&1
  echo "{\"prod\": $n}" >> gpurun_out/prod_ab2.jsonl
  timeout 300 python scripts/prefill_bench.py --no-cpu-baseline --configs p_prefix1,p_prefix5 >> gpurun_out/prod_ab2.jsonl 2>> gpurun_out/prod_ab2.err
  PA_PREFILL=3 timeout 300 python scripts/prefill_bench.py --no-cpu-baseline --configs p_sharegpt,p_2k >> gpurun_out/prod_ab2.jsonl 2>> gpurun_out/prod_ab2.err
done
