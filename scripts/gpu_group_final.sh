timeout 600 python -m pytest tests/test_gpu_grouped.py -m gpu -q 2>&1 | tail -1
for c in c5_beam c3_parallel c3_fork; do
  timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline --no-e2e --grouped -1 2>>gpurun_out/grouped.err
done > gpurun_out/bench_grouped_r01.jsonl
python -c "
import json
for l in open('gpurun_out/bench_grouped_r01.jsonl'):
    d=json.loads(l); print(d['config']['workload'], d['config']['decode_kernel'], round(d['us_per_step'],1), round(d['roofline']['frac'],3))"
