# Round evidence: tests, smoke, bench (default + all configs), ncu launch list + full capture.
TAG=${TAG:-r01}
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_${TAG}.txt; tail -3 gpurun_out/pytest_gpu_${TAG}.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; cat gpurun_out/smoke_${TAG}.txt
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; cat gpurun_out/bench_${TAG}.json
STEPS=500 bash scripts/bench_all.sh > gpurun_out/bench_all_${TAG}.jsonl
bash scripts/gpu_profile.sh c2_sharegpt $TAG
bash scripts/gpu_profile.sh c2_alpaca $TAG
bash scripts/gpu_profile.sh c5_beam $TAG
NCU_CFG="p_2k p_prefix5" TAG=$TAG bash scripts/gpu_prefill_bench.sh
