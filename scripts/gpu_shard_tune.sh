#!/bin/bash
# TP=8 rank-0 shard: stages / heads-per-CTA A/B (PA_STG, PA_HPC; scheduling only)
mkdir -p gpurun_out
rm -f gpurun_out/shard_tune.jsonl
for c in c2_sharegpt c2_alpaca; do
  for v in "0 0" "3 0" "4 0" "0 1" "3 1" "0 2" "3 5"; do
    set -- $v
    echo "{\"stg\": $1, \"hpc\": $2}" >> gpurun_out/shard_tune.jsonl
    PA_STG=$1 PA_HPC=$2 timeout 300 python bench.py --config $c --shard-of 8 --steps 500 --no-cpu-baseline --no-prefill --no-e2e >> gpurun_out/shard_tune.jsonl 2>> gpurun_out/shard_tune.err
  done
done
for g in 0 4; do
  echo "{\"c5_grouped\": $g}" >> gpurun_out/shard_tune.jsonl
  timeout 300 python bench.py --config c5_beam --shard-of 8 --grouped $g --steps 500 --no-cpu-baseline --no-prefill --no-e2e >> gpurun_out/shard_tune.jsonl 2>> gpurun_out/shard_tune.err
done
