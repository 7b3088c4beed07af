# partition size A/B (PA_PT) for coop on every config (attention alone, sweep.py)
for pt in 512 1024 2048 512 2048; do
  echo "== PA_PT=$pt"
  PA_PT=$pt SWEEP_SHAPES="coop,4,2,1" timeout 600 python scripts/sweep.py c2_sharegpt c3_parallel c3_fork c4_sharegpt c4_long c5_beam 2>&1 | grep -v Warn
done
