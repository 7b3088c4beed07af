#!/bin/bash
# Prefill (N4) benchmark + one ncu --set full capture of the prefill kernel (p_2k).
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 600 python scripts/prefill_bench.py > gpurun_out/prefill_bench_${TAG}.jsonl 2> gpurun_out/prefill_bench_${TAG}.err
cat gpurun_out/prefill_bench_${TAG}.jsonl
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_prefill -c 1 \
    -o gpurun_out/prefill_${TAG} python scripts/prefill_bench.py --configs ${NCU_CFG:-p_2k} --iters 1 \
    > gpurun_out/prefill_ncu_${TAG}.log 2>&1
  tail -3 gpurun_out/prefill_ncu_${TAG}.log
fi
