# scheduler A/B (device-timed bench lines, interleaved): SCHEDS="coop ncoop" CFGS="c2_alpaca c2_sharegpt"
SCHEDS=${SCHEDS:-"coop ncoop"}
CFGS=${CFGS:-"c2_alpaca c2_sharegpt"}
for rep in 1 2; do
  for s in $SCHEDS; do
    for c in $CFGS; do
      PA_SCHED=${s%%:*} PA_HPC=$(echo $s: | cut -d: -f2) timeout 300 python bench.py --config $c --steps 500 --warmup 10 --no-cpu-baseline --no-e2e 2>>gpurun_out/ab.err |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$s', d['config']['workload'], round(d['us_per_step'],1), round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['gpu_launches'])"
    done
  done
done
