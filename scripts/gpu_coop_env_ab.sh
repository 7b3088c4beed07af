#!/bin/bash
# env A/B of the coop decode kernel's CTA shape (PA_HPC heads per CTA, PA_STG stages) on C2
mkdir -p gpurun_out
rm -f gpurun_out/coop_env.jsonl
for env in "PA_HPC=4" "PA_HPC=4 PA_STG=3" "PA_HPC=2" "PA_HPC=2 PA_STG=6" "PA_HPC=8" "PA_HPC=4"; do
  for c in c2_alpaca c2_sharegpt; do
    echo "{\"env\": \"$env\"}" >> gpurun_out/coop_env.jsonl
    env $env timeout 150 python bench.py --config $c --no-cpu-baseline --no-prefill --no-e2e --steps 500 >> gpurun_out/coop_env.jsonl 2>> gpurun_out/coop_env.err
  done
done
