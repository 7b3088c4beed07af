#!/bin/bash
# exp2 emulation share A/B for the prompt kernels (PA_EXP_EMU = 0: all MUFU, k: every k-th pair on FMA)
mkdir -p gpurun_out
rm -f gpurun_out/emu_ab.jsonl
for n in 0 4 3 2; do
  make clean > /dev/null && make -j8 NVXFLAGS=-DPA_EXP_EMU=$n > gpurun_out/build_emu$n.txt 2>&1
  echo "{\"emu\": $n}" >> gpurun_out/emu_ab.jsonl
  timeout 300 python scripts/prefill_bench.py --no-cpu-baseline >> gpurun_out/emu_ab.jsonl 2>> gpurun_out/emu_ab.err
  PA_PREFILL=3 timeout 300 python scripts/prefill_bench.py --no-cpu-baseline --configs p_sharegpt,p_2k >> gpurun_out/emu_ab.jsonl 2>> gpurun_out/emu_ab.err
done
make clean > /dev/null && make -j8 > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/pytest_prefill.txt 2>&1; echo rc=$? >> gpurun_out/pytest_prefill.txt
make clean > /dev/null && make -j8 NVXFLAGS=-DPA_PREFILL_TRACE > gpurun_out/trace_build.txt 2>&1
timeout 300 python scripts/pf_trace.py p_prefix5 > gpurun_out/pf_trace.txt 2>&1
