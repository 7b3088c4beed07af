# grouped kernel: register caps 5-7 CTAs/SM x stages, one block slot per stage
for v in g5 g6 g7; do
  for st in 2 3 4; do
    PA_LIB_VARIANT=$v PA_GROUP_SLOTS=1 PA_GROUP_STG=$st timeout 300 python bench.py --config c5_beam --steps 300 --warmup 10 --no-cpu-baseline --no-e2e --no-prefill --grouped 4 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v stg=$st', d['config']['workload'], round(d['us_per_step'],1), round(d['roofline']['frac'],3))"
  done
done
for c in c3_fork c3_parallel; do
  PA_LIB_VARIANT=g6 PA_GROUP_SLOTS=1 timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline --no-e2e --no-prefill --grouped -1 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('g6 slots1', d['config']['workload'], round(d['us_per_step'],1), round(d['roofline']['frac'],3))"
done
