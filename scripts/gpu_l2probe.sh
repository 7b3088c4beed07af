#!/bin/bash
mkdir -p gpurun_out
make -j8 > gpurun_out/build.txt 2>&1
timeout 300 python scripts/tma_probe.py --l2 > gpurun_out/tma_probe_l2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/pytest_prefill.txt 2>&1; echo rc=$? >> gpurun_out/pytest_prefill.txt
