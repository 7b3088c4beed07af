#!/bin/bash
# prefill parity with a forced kernel variant + bench of that variant
V=$1
PA_PREFILL=$V timeout 600 python -m pytest tests/test_gpu_prefill.py -q -x 2>&1 | tail -3
PA_PREFILL=$V timeout 300 python scripts/prefill_bench.py --no-cpu-baseline 2>&1 | cut -c1-130
