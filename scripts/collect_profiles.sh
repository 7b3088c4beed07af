#!/bin/bash
# copy the evidence of a gpu_round.sh run (gpurun_out/, scratch) into profiles/ (tracked)
TAG=${TAG:-r01}
cp gpurun_out/bench_${TAG}.json profiles/${TAG}_bench.json
cp gpurun_out/bench_all_${TAG}.jsonl profiles/${TAG}_bench_all.jsonl
cp gpurun_out/prefill_bench_${TAG}.jsonl profiles/${TAG}_prefill_bench.jsonl
cp gpurun_out/pytest_gpu_${TAG}.txt profiles/${TAG}_pytest_gpu.txt
cp gpurun_out/smoke_${TAG}.txt profiles/${TAG}_smoke.txt
for c in c2_sharegpt c2_alpaca c5_beam; do
  cp gpurun_out/launches_${c}_${TAG}.csv profiles/launches_${c}_${TAG}.csv
  ncu -i gpurun_out/prof_attn_${c}_${TAG}.ncu-rep --page details > profiles/${TAG}_${c}_attention_ncu_details.txt 2>/dev/null
done
for c in p_2k p_prefix5; do
  ncu -i gpurun_out/prefill_${TAG}_${c}.ncu-rep --page details > profiles/${TAG}_prefill_${c}_ncu_details.txt 2>/dev/null
done
ls -la profiles
python scripts/ncu_traffic.py ${TAG} c2_sharegpt c2_alpaca c5_beam
