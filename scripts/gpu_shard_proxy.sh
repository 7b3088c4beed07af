#!/bin/bash
# Per-rank kernel time of TP = 2/4/8 (rank 0's head shard on one GPU, no exchange)
mkdir -p gpurun_out
rm -f gpurun_out/shard_proxy.jsonl
for c in c2_sharegpt c2_alpaca c4_long c5_beam; do
  for P in 2 4 8; do
    timeout 300 python bench.py --config $c --shard-of $P --steps 500 --no-cpu-baseline --no-prefill --no-e2e >> gpurun_out/shard_proxy.jsonl 2>> gpurun_out/shard_proxy.err
  done
done
