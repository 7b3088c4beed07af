#!/bin/bash
# ncu --set full of the tcgen05 N1 decode (bench.py default) on c5_beam and c3_fork, plus
# the launch lists of both default bench commands
mkdir -p gpurun_out/n1prof
for cfg in c5_beam c3_fork; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:group_tc -s 8 -c 1 -o gpurun_out/n1prof/$cfg \
      python bench.py --config $cfg --steps 3 --warmup 8 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/n1prof/$cfg.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 40 --csv --log-file gpurun_out/n1prof/launches_$cfg.csv \
      python bench.py --config $cfg --steps 20 --warmup 10 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/n1prof/launches_$cfg.log 2>&1
done
