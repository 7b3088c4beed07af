#!/bin/bash
mkdir -p gpurun_out
make clean > /dev/null && make -j8 NVXFLAGS=-DPA_TC_TRACE > gpurun_out/trace_build.txt 2>&1
timeout 300 python scripts/tc_trace.py c5_beam 4 > gpurun_out/tc_trace_c5.txt 2>&1
make clean > /dev/null && make -j8 > gpurun_out/build.txt 2>&1
