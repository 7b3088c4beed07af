#!/bin/bash
# e2e (pa_decode_step) chunk-weight sweep (PA_E2E_SPLIT) + host-API parity under a split
PA_E2E_SPLIT=1,2,4,1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "decode_step" 2>&1 | tail -2
for rep in 1 2; do
for sp in ${SPLITS:-"1,1,1,1" "1,3,3,1" "1,2,4,1" "1,2,4,4,1" "1,2,3,3,2,1" "1,2,4,8,2" "1,2,2,2,1"}; do
  PA_E2E_SPLIT=$sp timeout 300 python bench.py --config ${CFG:-c2_sharegpt} --steps 200 --no-cpu-baseline --no-prefill > gpurun_out/e2e_sp.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_sp.json')); print('split $sp', round(d['e2e']['value']), round(d['e2e']['ms_per_step']*1e3,1), 'host', d['e2e'].get('host_enqueue_us_per_step'), 'dev', round(d['us_per_step'],1))"
done
done
