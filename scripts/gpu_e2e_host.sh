for st in 1 2; do for ch in 1 2 4; do
  PA_E2E_STREAMS=$st PA_E2E_CHUNKS=$ch timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/e2eh_${st}_${ch}.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2eh_${st}_${ch}.json')); print('streams $st chunks $ch value', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step']*1e3,1), 'host', d['e2e']['host_enqueue_us_per_step'])"
done; done
