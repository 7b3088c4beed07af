# One bench line per BASELINE config (device-timed; no cpu baseline / e2e).
STEPS=${STEPS:-300}
for c in c2_sharegpt c2_alpaca c3_parallel c3_fork c4_sharegpt c4_long c5_beam c1_tiny; do
  timeout 300 python bench.py --config $c --steps $STEPS --warmup 10 --no-cpu-baseline --no-e2e "$@" 2>>gpurun_out/bench_all.err
done
