# grouped (tensor-core N1) kernel: leader search by match.any (variant gm) vs shuffle loop
timeout 600 python -m pytest tests/test_gpu_grouped.py -m gpu -q -x 2>&1 | tail -1
for v in gm cur gm cur; do
  if [ $v = cur ]; then LV=""; else LV=$v; fi
  for c in c5_beam c3_fork; do
    PA_LIB_VARIANT=$LV timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline --no-e2e --grouped -1 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['workload'], d['config']['decode_kernel'], round(d['us_per_step'],1), round(d['roofline']['frac'],3))"
  done
done
