# shared kernel: register cap for 4 CTAs/SM (variant mb4, 56 regs) vs default (72 regs, 3 CTAs/SM)
for v in cur mb4 cur mb4; do
  if [ $v = cur ]; then LV=""; else LV=$v; fi
  echo "== $v"
  PA_LIB_VARIANT=$LV SWEEP_SHAPES="shared4,2,3,1;shared4,2,4,1;shared4,1,4,1;shared4,1,6,1" timeout 300 python scripts/sweep.py c5_beam 2>&1 | grep -v Warn
done
