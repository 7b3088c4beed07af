#!/bin/bash
# compare a variant build (PA_LIB_VARIANT=$V) with the default on the prefill parity tests + bench
V=$1
for lib in "" "$V"; do
  echo "== variant '${lib:-default}'"
  export PA_LIB_VARIANT=$lib
  timeout 600 python -m pytest tests/test_gpu_prefill.py -q -x 2>&1 | tail -2
  timeout 300 python scripts/prefill_bench.py --no-cpu-baseline 2>&1 | cut -c1-130
done
