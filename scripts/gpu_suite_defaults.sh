mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
rm -f gpurun_out/defaults.jsonl
for c in c5_beam c3_fork c3_parallel; do timeout 200 python bench.py --config $c --no-cpu-baseline --no-prefill --no-e2e >> gpurun_out/defaults.jsonl 2>>gpurun_out/defaults.err; done
