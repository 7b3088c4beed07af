#!/bin/bash
# one iteration on the tcgen05 N1 decode: its GPU tests, then bench lines on C5 / C3
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_grouped.py -q -x > gpurun_out/pytest_grouped.txt 2>&1; rc=$?; echo rc=$rc >> gpurun_out/pytest_grouped.txt
[ $rc -ne 0 ] && exit 1
rm -f gpurun_out/tc_bench.jsonl
for c in "c5_beam --grouped 4" "c3_fork --grouped 6" "c3_parallel --grouped 6"; do
  timeout 150 python bench.py --config $c --no-cpu-baseline --no-prefill --no-e2e --steps 300 >> gpurun_out/tc_bench.jsonl 2>> gpurun_out/tc_bench.err
  PA_TC_SPLIT=0 timeout 150 python bench.py --config $c --no-cpu-baseline --no-prefill --no-e2e --steps 300 >> gpurun_out/tc_bench.jsonl 2>> gpurun_out/tc_bench.err
done
