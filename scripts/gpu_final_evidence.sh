# Final round evidence after the N1 change: tests, smoke, default bench, bench_all.
TAG=${TAG:-r01}
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_${TAG}.txt; tail -2 gpurun_out/pytest_gpu_${TAG}.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; cat gpurun_out/smoke_${TAG}.txt
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; cut -c1-300 gpurun_out/bench_${TAG}.json
STEPS=500 bash scripts/bench_all.sh > gpurun_out/bench_all_${TAG}.jsonl
timeout 300 python bench.py --config c5_beam --steps 500 --warmup 10 --no-cpu-baseline --no-e2e --shared 0 >> gpurun_out/bench_all_${TAG}.jsonl 2>>gpurun_out/bench_all.err
python - <<'PY'
import json
for l in open("gpurun_out/bench_all_r01.jsonl"):
    d = json.loads(l); r = d["roofline"]
    print(d["config"]["workload"], d["config"]["decode_kernel"], round(d["us_per_step"], 1), round(r["frac"], 3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
