#!/bin/bash
# the two-tile packed prompt kernel (v7): prompt tests, then the prompt bench with v7 and the v6 ablation
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/pytest_prefill.txt 2>&1; rc=$?; echo rc=$rc >> gpurun_out/pytest_prefill.txt
[ $rc -ne 0 ] && exit 1
rm -f gpurun_out/pf_v7.jsonl
for v in 7 6 7; do
  echo "{\"packed\": $v}" >> gpurun_out/pf_v7.jsonl
  PA_PACKED=$v timeout 300 python scripts/prefill_bench.py --no-cpu-baseline --configs p_prefix5,p_prefix1 >> gpurun_out/pf_v7.jsonl 2>> gpurun_out/pf_v7.err
done
