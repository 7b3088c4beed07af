#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tp_fused.py tests/test_bench_contract.py -m gpu -q > gpurun_out/pytest_tp.txt 2>&1; echo rc=$? >> gpurun_out/pytest_tp.txt
for c in c2_sharegpt c2_alpaca; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-prefill >> gpurun_out/bench_r02a.jsonl 2>> gpurun_out/bench_r02a.err; done
