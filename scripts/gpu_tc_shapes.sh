#!/bin/bash
# tcgen05 N1 kernel: pieces per tile x tile buffers (same shared memory budget), c5 / c3_fork
mkdir -p gpurun_out
rm -f gpurun_out/tc_shapes.jsonl
for v in "2 3" "1 6" "1 5" "1 4"; do
  set -- $v
  make clean > /dev/null && make -j8 NVXFLAGS="-DPA_TC_SLOTS=$1 -DPA_TC_BUF=$2" > /dev/null 2>&1
  for c in c5_beam "c3_fork --grouped 6"; do
    echo "{\"slots\": $1, \"bufs\": $2}" >> gpurun_out/tc_shapes.jsonl
    timeout 300 python bench.py --config $c --steps 300 --no-cpu-baseline --no-prefill --no-e2e >> gpurun_out/tc_shapes.jsonl 2>> gpurun_out/tc_shapes.err
  done
done
timeout 300 python -m pytest tests/test_gpu_grouped.py -q -x > gpurun_out/pytest_grouped_shapes.txt 2>&1
make clean > /dev/null && make -j8 > /dev/null 2>&1
