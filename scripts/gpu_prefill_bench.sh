#!/bin/bash
# Prefill (N4) benchmark + ncu --set full captures of the prefill kernel.
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 600 python scripts/prefill_bench.py > gpurun_out/prefill_bench_${TAG}.jsonl 2> gpurun_out/prefill_bench_${TAG}.err
cat gpurun_out/prefill_bench_${TAG}.jsonl
if [ "${NCU:-1}" = "1" ]; then
  for cfg in ${NCU_CFG:-p_2k}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_prefill -c 1 \
      -o gpurun_out/prefill_${TAG}_${cfg} -f python scripts/prefill_bench.py --configs $cfg --iters 1 \
      > gpurun_out/prefill_ncu_${TAG}_${cfg}.log 2>&1
    tail -2 gpurun_out/prefill_ncu_${TAG}_${cfg}.log
  done
fi
