#!/bin/bash
# per-tile clock64 trace of the tcgen05 N1 decode (variant build), then the normal build back
mkdir -p gpurun_out
make clean > /dev/null && make -j8 NVXFLAGS=-DPA_TC_TRACE > gpurun_out/trace_build.txt 2>&1
TC_TRACE_CACHES=3 timeout 180 python scripts/tc_trace.py c5_beam 4 > gpurun_out/tc_trace_c5.txt 2>&1
TC_TRACE_CACHES=4 timeout 180 python scripts/tc_trace.py c3_fork 6 > gpurun_out/tc_trace_c3f.txt 2>&1
make clean > /dev/null && make -j8 > gpurun_out/build.txt 2>&1
