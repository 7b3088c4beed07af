#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=15 > gpurun_out/pytest_gpu.txt 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
for c in c2_sharegpt c2_alpaca; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-prefill >> gpurun_out/bench_r02b.jsonl 2>> gpurun_out/bench_r02b.err; done
