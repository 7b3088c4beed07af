#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --config c5_beam --grouped 4 --no-cpu-baseline --no-prefill --no-e2e --steps 300 >> gpurun_out/bench_r02f.jsonl 2>> gpurun_out/bench_r02f.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:group_tc -s 5 -c 1 -o gpurun_out/c5_grouped_tc python bench.py --config c5_beam --grouped 4 --steps 3 --warmup 5 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/ncu_c5g.log 2>&1
