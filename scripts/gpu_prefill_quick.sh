#!/bin/bash
# quick prefill check: parity tests + bench + trace
rm -f gpurun_out/prefill_tests.log
bash scripts/gpu_prefill.sh > /dev/null 2>&1; grep exit gpurun_out/prefill_tests.log | tr '\n' ' '; echo
grep -h "assert\|Error\|error" gpurun_out/prefill_tests.log | head -5
timeout 300 python scripts/prefill_bench.py 2>&1 | cut -c1-170
