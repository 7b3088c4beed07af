#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/pytest_prefill.txt 2>&1; echo rc=$? >> gpurun_out/pytest_prefill.txt
timeout 600 python scripts/prefill_bench.py --no-cpu-baseline > gpurun_out/prefill_bench_r02.jsonl 2> gpurun_out/prefill_bench_r02.err
