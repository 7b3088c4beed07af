#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/ablate.py order c2_alpaca c2_sharegpt > gpurun_out/ablate_order.jsonl 2>&1
timeout 600 python scripts/ablate.py block_size c2_sharegpt c2_alpaca > gpurun_out/ablate_bs.jsonl 2>&1
timeout 600 python scripts/ablate.py placement c2_sharegpt c2_alpaca > gpurun_out/ablate_pl.jsonl 2>&1
timeout 300 python bench.py --config c2_alpaca --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/bench_c2a.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attention_coop -s 20 -c 1 -o gpurun_out/c2a_r02 python bench.py --config c2_alpaca --steps 5 --warmup 20 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/ncu_c2a.log 2>&1
