#!/bin/bash
# one iteration on the prompt kernels: their GPU tests, the prompt bench, the packed-kernel trace
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/pytest_prefill.txt 2>&1; rc=$?; echo rc=$rc >> gpurun_out/pytest_prefill.txt
[ $rc -ne 0 ] && exit 1
timeout 600 python scripts/prefill_bench.py --no-cpu-baseline > gpurun_out/prefill_bench.jsonl 2> gpurun_out/prefill_bench.err
bash scripts/gpu_pf_trace.sh
