#!/bin/bash
# env A/B of the tcgen05 N1 decode's split context (PA_TC_PART / PA_TC_SPLIT) + its tests under both
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_grouped.py -q -x > gpurun_out/pytest_grouped.txt 2>&1; echo rc=$? >> gpurun_out/pytest_grouped.txt
PA_TC_SPLIT=2 timeout 300 python -m pytest tests/test_gpu_grouped.py -q -x > gpurun_out/pytest_grouped_split2.txt 2>&1; echo rc=$? >> gpurun_out/pytest_grouped_p256.txt
rm -f gpurun_out/tc_env.jsonl
for env in "PA_TC_SPLIT=1" "PA_TC_SPLIT=0" "PA_TC_SPLIT=2"; do
  for c in "c5_beam --grouped 4" "c3_fork --grouped 6" "c3_parallel --grouped 6"; do
    echo "{\"env\": \"$env\"}" >> gpurun_out/tc_env.jsonl
    env $env timeout 150 python bench.py --config $c --no-cpu-baseline --no-prefill --no-e2e --steps 300 >> gpurun_out/tc_env.jsonl 2>> gpurun_out/tc_env.err
  done
done
