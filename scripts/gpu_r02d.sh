#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tp_fused.py tests/test_bench_contract.py -m gpu -q -x > gpurun_out/pytest_d.txt 2>&1; echo rc=$? >> gpurun_out/pytest_d.txt
for c in c2_alpaca c2_sharegpt c4_long c3_parallel; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-prefill >> gpurun_out/bench_r02d.jsonl 2>> gpurun_out/bench_r02d.err
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-prefill --no-e2e --no-plan >> gpurun_out/bench_r02d_noplan.jsonl 2>> gpurun_out/bench_r02d.err
done
