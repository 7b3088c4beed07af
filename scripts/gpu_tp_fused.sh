#!/bin/bash
# N2 fused TP all-gather tests on one GPU (simulated ranks + 2 processes over CUDA IPC)
timeout 600 python -m pytest tests/test_gpu_tp_fused.py -q -x 2>&1 | tail -15
