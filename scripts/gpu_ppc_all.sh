# coop partitions-per-CTA (scheduling only, bitwise identical) vs PT=2048 on every config
SWEEP_SHAPES="coop,4,2,1;coop,4,2,4;coop,4,2,2" timeout 600 python scripts/sweep.py c2_sharegpt c3_parallel c4_sharegpt c4_long c5_beam 2>&1 | grep -v Warn
PA_PT=2048 SWEEP_SHAPES="coop,4,2,1" timeout 600 python scripts/sweep.py c2_sharegpt c3_parallel c4_sharegpt c4_long c5_beam 2>&1 | grep -v Warn
SWEEP_SHAPES="shared4,2,3,1;shared4,2,3,4" timeout 600 python scripts/sweep.py c5_beam 2>&1 | grep -v Warn
