# pa_decode_step transfer modes: parity tests, then the bench e2e number per mode; library comparison
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k decode_step 2>&1 | tail -3
for st in 1 2; do for ch in 4 6 8 12; do
  PA_E2E_STREAMS=$st PA_E2E_CHUNKS=$ch timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/e2e_${st}_${ch}.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_${st}_${ch}.json')); print('streams $st chunks $ch value', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step']*1e3,1))"
done; done
timeout 900 python scripts/compare_libs.py c2_sharegpt c2_alpaca c4_long c5_beam > gpurun_out/compare_libs.jsonl 2> gpurun_out/compare_libs.err
tail -5 gpurun_out/compare_libs.err
cat gpurun_out/compare_libs.jsonl
