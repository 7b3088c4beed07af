#!/bin/bash
# prefill parity then benchmark (no ncu)
rm -f gpurun_out/prefill_tests.log
bash scripts/gpu_prefill.sh
NCU=${NCU:-0} bash scripts/gpu_prefill_bench.sh
