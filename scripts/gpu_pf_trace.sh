#!/bin/bash
# per-item timeline of the packed prompt kernel (variant build), then the normal build back
mkdir -p gpurun_out
make clean > /dev/null && make -j8 NVXFLAGS=-DPA_PREFILL_TRACE > gpurun_out/pf_trace_build.txt 2>&1
timeout 300 python scripts/pf_trace.py p_prefix5 > gpurun_out/pf_trace.txt 2>&1
timeout 300 python scripts/pf_trace.py p_prefix1 >> gpurun_out/pf_trace.txt 2>&1
make clean > /dev/null && make -j8 > gpurun_out/build.txt 2>&1
