# A/B of the current libpagedattn.so against a baseline variant (libpagedattn_base.so),
# interleaved, device-timed bench lines; then a coop launch-shape sweep.
#   V=base CFGS="c2_alpaca c2_sharegpt" bash scripts/gpu_ab.sh
V=${V:-base}
CFGS=${CFGS:-"c2_alpaca c2_sharegpt c4_sharegpt c5_beam"}
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
for rep in 1 2; do
  for v in $V cur; do
    for c in $CFGS; do
      if [ $v = cur ]; then LV=""; else LV=$v; fi
      PA_LIB_VARIANT=$LV timeout 300 python bench.py --config $c --steps 500 --warmup 10 --no-cpu-baseline --no-e2e 2>>gpurun_out/ab.err |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['workload'], round(d['us_per_step'],1), round(d['roofline']['achieved']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    done
  done
done
if [ -n "$SWEEP_SHAPES" ]; then
  timeout 900 python scripts/sweep.py $SWEEP_CFGS 2>>gpurun_out/ab.err
fi
