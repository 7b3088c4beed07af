#!/bin/bash
# e2e (pa_decode_step) chunk-count sweep + the host-API parity test
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "decode_step" 2>&1 | tail -2
for c in ${CHUNKS:-1 2 3 4}; do
  PA_E2E_CHUNKS=$c timeout 300 python bench.py --steps 200 --no-cpu-baseline --no-prefill > gpurun_out/e2e_$c.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_$c.json')); print('chunks $c', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],4), round(d['value']))"
done
