#!/bin/bash
# e2e (pa_decode_step): captured-graph replay vs eager enqueue, and chunk weights
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "decode_step" 2>&1 | tail -2
for rep in ${REPS:-1 2}; do
for g in 1 0; do
for sp in ${SPLITS:-"1,1,1,1" "1,2,4,4,1" "1,2,4,1" "1,1,1,1,1,1"}; do
  PA_E2E_GRAPH=$g PA_E2E_SPLIT=$sp timeout 300 python bench.py --config ${CFG:-c2_sharegpt} --steps 200 --no-cpu-baseline --no-prefill > gpurun_out/e2e_g.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_g.json')); print('graph $g split $sp', round(d['e2e']['value']), round(d['e2e']['ms_per_step']*1e3,1), 'host', d['e2e'].get('host_enqueue_us_per_step'), 'dev', round(d['us_per_step'],1))"
done
done
done
