#!/bin/bash
# one iteration on the prompt kernels: tests + bench on the normal build, then the v6 trace
mkdir -p gpurun_out
make clean > /dev/null && make -j8 > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/pytest_prefill.txt 2>&1; echo rc=$? >> gpurun_out/pytest_prefill.txt
timeout 600 python scripts/prefill_bench.py --no-cpu-baseline > gpurun_out/prefill_bench.jsonl 2> gpurun_out/prefill_bench.err
PA_PREFILL=3 timeout 600 python scripts/prefill_bench.py --no-cpu-baseline --configs p_sharegpt,p_2k,p_chunk256 > gpurun_out/prefill_bench_v3.jsonl 2>> gpurun_out/prefill_bench.err
make clean > /dev/null && make -j8 NVXFLAGS=-DPA_PREFILL_TRACE > gpurun_out/trace_build.txt 2>&1
timeout 300 python scripts/pf_trace.py p_prefix5 > gpurun_out/pf_trace.txt 2>&1
