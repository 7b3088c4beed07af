for v in cur h5 h6; do
  if [ $v = cur ]; then LV=""; else LV=$v; fi
  for st in 2 3; do
    PA_LIB_VARIANT=$LV PA_GROUP_HG=2 PA_GROUP_STG=$st timeout 300 python bench.py --config c5_beam --steps 300 --warmup 10 --no-cpu-baseline --no-e2e --no-prefill --grouped -1 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v stg=$st', d['config']['workload'], round(d['us_per_step'],1), round(d['roofline']['frac'],3))"
  done
done
