#!/bin/bash
mkdir -p gpurun_out
make clean > /dev/null && make -j8 NVXFLAGS=-DPA_PREFILL_TRACE > gpurun_out/trace_build.txt 2>&1
timeout 300 python scripts/pf_trace.py p_prefix5 > gpurun_out/pf_trace.txt 2>&1
timeout 300 python scripts/pf_trace.py p_prefix1 >> gpurun_out/pf_trace.txt 2>&1
