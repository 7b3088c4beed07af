mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_tp_fused.py -q -x > gpurun_out/pytest_stg1.txt 2>&1; echo rc=$? >> gpurun_out/pytest_stg1.txt
rm -f gpurun_out/stg1.jsonl
for c in c2_alpaca c1_tiny c2_sharegpt; do timeout 200 python bench.py --config $c --no-cpu-baseline --no-prefill >> gpurun_out/stg1.jsonl 2>>gpurun_out/stg1.err; done
