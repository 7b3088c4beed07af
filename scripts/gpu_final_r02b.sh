#!/bin/bash
# Round-2 closing evidence on the final tree: GPU suite, smoke, sanitizers on the tcgen05 N1
# kernel, the default bench line (CPU baseline + N4 context line + read probe), every
# config's line, the reference arm, the prompt-kernel bench, and the ncu launch lists of
# the default command, c5_beam and c3_fork (our kernels only: -k regex)
D=gpurun_out/final
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $D/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $D/pytest_gpu.txt 2>&1; echo "rc=$?" >> $D/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; echo "smoke rc=$?" >> $D/smoke.txt
for tool in memcheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 3 python scripts/sanitize_grouped.py > $D/sanitize_grouped_$tool.txt 2>&1; echo "rc=$?" >> $D/sanitize_grouped_$tool.txt
done
timeout 900 python bench.py > $D/bench_default.jsonl 2> $D/bench_default.err
for c in c2_alpaca c3_parallel c3_fork c4_sharegpt c4_long c5_beam c1_tiny; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-prefill >> $D/bench_all.jsonl 2>> $D/bench_all.err
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $D/bench_reference.jsonl 2> $D/bench_reference.err
timeout 600 python scripts/prefill_bench.py > $D/prefill_bench.jsonl 2> $D/prefill_bench.err
K='regex:paged_attention|copy_blocks|reshape_and_cache|group_tc|tp_signal'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file $D/launches_c2_sharegpt.csv \
    python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-prefill --no-e2e > $D/launches_c2_sharegpt.log 2>&1
for c in c5_beam c3_fork; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file $D/launches_$c.csv \
      python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-prefill --no-e2e > $D/launches_$c.log 2>&1
done
