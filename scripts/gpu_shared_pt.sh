# partition size A/B (PA_PT) for the shared kernel on c5 and coop on c5 / c2
for pt in 512 768 1024 2048 512; do
  echo "== PA_PT=$pt"
  PA_PT=$pt SWEEP_SHAPES="coop,4,2,1;shared4,2,3,1" timeout 300 python scripts/sweep.py c5_beam 2>&1 | grep -v Warn
done
