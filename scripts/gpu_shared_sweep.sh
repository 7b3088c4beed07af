# N1 CUDA-core sharing-aware decode: stage-stream variants (heads per CTA, slots per stage,
# stages) against coop on the sharing configs; parity tests; bench lines coop vs shared.
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
# fields: sched, heads per CTA, stages, slots per stage (shared) / partitions per CTA (coop)
SWEEP_SHAPES="coop,4,2,1;shared4,2,3,1;shared4,2,4,1;shared4,2,5,1;shared4,1,4,1;shared4,1,6,1;shared4,1,8,1;shared4,2,2,2" \
  timeout 900 python scripts/sweep.py c5_beam 2>&1 | grep -v Warn
SWEEP_SHAPES="coop,4,2,1;shared6,1,4,1;shared6,1,8,1;shared6,1,3,2;shared6,1,2,3;shared3,2,4,1" \
  timeout 900 python scripts/sweep.py c3_parallel c3_fork 2>&1 | grep -v Warn
for c in c5_beam c3_fork c3_parallel; do
  for sh in 0 $( [ $c = c5_beam ] && echo 4 || echo 6 ); do
    timeout 300 python bench.py --config $c --steps 500 --warmup 10 --no-cpu-baseline --no-e2e --shared $sh 2>>gpurun_out/sh.err |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('shared=$sh', d['config']['workload'], round(d['us_per_step'],1), round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
