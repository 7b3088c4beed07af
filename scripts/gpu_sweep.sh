set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt; cat gpurun_out/pytest_gpu.txt
STEPS=300 bash scripts/bench_all.sh > gpurun_out/bench_all.jsonl
STEPS=300 bash scripts/bench_all.sh --unfused > gpurun_out/bench_all_unfused.jsonl
