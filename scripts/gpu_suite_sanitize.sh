#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=10 > gpurun_out/pytest_gpu.txt 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
for tool in memcheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 3 python scripts/sanitize_grouped.py > gpurun_out/sanitize_grouped_$tool.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitize_grouped_$tool.txt
done
rm -f gpurun_out/bench_h.jsonl
for c in c5_beam c3_fork c3_parallel; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-prefill >> gpurun_out/bench_h.jsonl 2>> gpurun_out/bench_h.err; done
