set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt; cat gpurun_out/pytest_gpu.txt
STEPS=300 bash scripts/bench_all.sh > gpurun_out/bench_all.jsonl
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
bash scripts/gpu_profile.sh c2_sharegpt r01c
