#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/tma_probe.py > gpurun_out/tma_probe.txt 2>&1
