#!/bin/bash
# TMA producer-warp count A/B for the prefill kernels (v3 / v6): PA_PF_PROD = 1, 2, 4
mkdir -p gpurun_out
rm -f gpurun_out/prod_ab.jsonl
for n in 1 2 4; do
  make clean > /dev/null && make -j8 NVXFLAGS=-DPA_PF_PROD=$n > gpurun_out/build_prod$n.txt 2>&1
  for v in 0 3; do
    echo "{\"prod\": $n, \"PA_PREFILL\": $v}" >> gpurun_out/prod_ab.jsonl
    PA_PREFILL=$v timeout 300 python scripts/prefill_bench.py --no-cpu-baseline >> gpurun_out/prod_ab.jsonl 2>> gpurun_out/prod_ab.err
  done
done
make clean > /dev/null && make -j8 > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/pytest_prefill.txt 2>&1; echo rc=$? >> gpurun_out/pytest_prefill.txt
