# grouped kernel: 2 heads per CTA (PA_GROUP_HG=2) vs 1: parity tests, then c5 / c3 bench lines
timeout 600 env PA_GROUP_HG=2 python -m pytest tests/test_gpu_grouped.py -m gpu -q -x 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_grouped.py -m gpu -q -x 2>&1 | tail -1
for hg in 1 2 1 2; do for c in c5_beam c3_fork; do
  PA_GROUP_HG=$hg timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline --no-e2e --no-prefill --grouped -1 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hg=$hg', d['config']['workload'], round(d['us_per_step'],1), round(d['roofline']['frac'],3))"
done; done
