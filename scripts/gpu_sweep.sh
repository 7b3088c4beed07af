timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python scripts/sweep.py c2_sharegpt c2_alpaca c4_long c5_beam c3_parallel > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
tail -3 gpurun_out/sweep.err
