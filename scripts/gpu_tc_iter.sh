#!/bin/bash
# one iteration on the tcgen05 grouped decode: traced build -> timeline; normal build -> tests + bench lines
mkdir -p gpurun_out
make clean > /dev/null && make -j8 NVXFLAGS=-DPA_TC_TRACE > gpurun_out/trace_build.txt 2>&1
timeout 300 python scripts/tc_trace.py c5_beam 4 > gpurun_out/tc_trace_c5.txt 2>&1
make clean > /dev/null && make -j8 > gpurun_out/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_grouped.py -q -x > gpurun_out/pytest_grouped.txt 2>&1; echo rc=$? >> gpurun_out/pytest_grouped.txt
rm -f gpurun_out/bench_tc.jsonl
for c in "c5_beam --grouped 4" "c3_fork --grouped 6" "c3_parallel --grouped 6"; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-prefill --no-e2e --steps 300 >> gpurun_out/bench_tc.jsonl 2>> gpurun_out/bench_tc.err
done
