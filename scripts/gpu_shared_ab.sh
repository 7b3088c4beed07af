# A/B of the shared producer variants (block-id prefetch, match.any leaders)
for v in base nomatch nopref cur base cur; do
  if [ $v = cur ]; then LV=""; else LV=$v; fi
  echo "== $v"
  PA_LIB_VARIANT=$LV SWEEP_SHAPES="shared4,2,4,1;shared4,1,4,1" timeout 300 python scripts/sweep.py c5_beam 2>&1 | grep -v Warn
done
