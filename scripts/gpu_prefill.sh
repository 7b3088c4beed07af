#!/bin/bash
# Prefill (N4) parity on the GPU, each test under its own timeout.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm --format=csv > gpurun_out/prefill_gpu.txt 2>&1
for t in test_degenerate_cases test_prompt_phase_vs_oracle test_shared_prefix_suffix_vs_oracle \
         test_block_size_and_placement_invariance_bitwise test_chunked_prompt_equals_whole_prompt_bitwise \
         test_prefill_sharegpt_sized_sampled_rows test_kernel_variants_agree; do
  timeout 300 python -m pytest tests/test_gpu_prefill.py -q -x -k "$t" >> gpurun_out/prefill_tests.log 2>&1
  echo "$t exit $?" >> gpurun_out/prefill_tests.log
done
tail -5 gpurun_out/prefill_tests.log
grep exit gpurun_out/prefill_tests.log
