for v in cur s5 cur s5; do
  if [ $v = cur ]; then LV=""; else LV=$v; fi
  echo "== $v"
  PA_LIB_VARIANT=$LV SWEEP_SHAPES="shared4,2,2,1;shared4,2,3,1" timeout 300 python scripts/sweep.py c5_beam 2>&1 | grep -v Warn
done
