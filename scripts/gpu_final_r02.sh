#!/bin/bash
# Round-2 bench lines for every config (default flags), the headline line with the CPU
# baseline, the reference arm, and the ncu launch list of the default bench command
mkdir -p gpurun_out/r02final
D=gpurun_out/r02final
timeout 900 python bench.py > $D/bench_default.jsonl 2> $D/bench_default.err
for c in c2_alpaca c3_parallel c3_fork c4_sharegpt c4_long c5_beam c1_tiny; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-prefill >> $D/bench_all.jsonl 2>> $D/bench_all.err
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $D/bench_reference.jsonl 2> $D/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"paged_attention|copy_blocks|reshape_and_cache|group_tc|tp_signal" \
    --csv --log-file $D/launches_default.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-prefill --no-e2e > $D/launches_default.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"paged_attention|copy_blocks|reshape_and_cache|group_tc" \
    --csv --log-file $D/launches_c5.csv python bench.py --config c5_beam --steps 20 --warmup 5 --no-cpu-baseline --no-prefill --no-e2e > $D/launches_c5.log 2>&1
