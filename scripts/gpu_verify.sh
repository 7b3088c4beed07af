# Quick verification of the current tree: GPU tests, smoke, default bench line.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_verify.txt; tail -3 gpurun_out/pytest_gpu_verify.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_verify.txt 2>&1; cat gpurun_out/smoke_verify.txt
timeout 600 python bench.py > gpurun_out/bench_verify.json 2> gpurun_out/bench_verify.err; cat gpurun_out/bench_verify.json
