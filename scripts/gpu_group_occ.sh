# grouped (tensor-core N1) kernel occupancy: register caps (variants g6: 6 CTAs/SM, g8: 8) x block slots per stage
timeout 600 env PA_LIB_VARIANT=g8 python -m pytest tests/test_gpu_grouped.py -m gpu -q -x 2>&1 | tail -1
for v in cur g6 g8; do
  if [ $v = cur ]; then LV=""; else LV=$v; fi
  for sl in 2 1; do
    PA_LIB_VARIANT=$LV PA_GROUP_SLOTS=$sl timeout 300 python bench.py --config c5_beam --steps 300 --warmup 10 --no-cpu-baseline --no-e2e --no-prefill --grouped 4 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v slots=$sl', d['config']['workload'], round(d['us_per_step'],1), round(d['roofline']['frac'],3))"
  done
done
