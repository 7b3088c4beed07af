# Round evidence for the final tree: gpu_round.sh + grouped (N1) lines + reference arm.
TAG=${TAG:-r01}
bash scripts/gpu_round.sh
for c in c5_beam c3_parallel c3_fork; do
  timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline --no-e2e --grouped -1 2>>gpurun_out/grouped.err
done > gpurun_out/bench_grouped_${TAG}.jsonl
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference_${TAG}.json 2>gpurun_out/reference.err
tail -c 600 gpurun_out/bench_reference_${TAG}.json
