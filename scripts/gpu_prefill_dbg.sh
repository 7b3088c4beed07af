#!/bin/bash
for B in 16 128; do for d in 0 3; do echo "B=$B debug=$d"; PA_PREFILL_DEBUG=$d timeout 300 python scripts/prefill_bench.py --configs ${CFGS:-p_2k,p_prefix5} --block-size $B 2>&1 | cut -c1-150; done; done
