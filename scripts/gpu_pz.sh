# coop grid order A/B: partition index fastest (default) vs slowest (PA_PZ=1); bench step lines
timeout 600 env PA_PZ=1 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
for rep in 1 2; do for pz in 0 1; do
  echo "== PA_PZ=$pz"
  PA_PZ=$pz SWEEP_SHAPES="coop,4,2,1" timeout 600 python scripts/sweep.py c2_sharegpt c2_alpaca c3_parallel c4_sharegpt c4_long c5_beam 2>&1 | grep -v Warn
done; done
for pz in 0 1 0 1; do
  PA_PZ=$pz timeout 300 python bench.py --config c2_sharegpt --steps 500 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench PA_PZ=$pz', d['config']['workload'], round(d['us_per_step'],1), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
