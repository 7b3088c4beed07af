#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_grouped.py -q -x > gpurun_out/pytest_grouped.txt 2>&1; echo rc=$? >> gpurun_out/pytest_grouped.txt
for c in "c5_beam --grouped 4" "c3_fork --grouped 6" "c3_parallel --grouped 6"; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-prefill --no-e2e --steps 300 >> gpurun_out/bench_r02g.jsonl 2>> gpurun_out/bench_r02g.err
done
