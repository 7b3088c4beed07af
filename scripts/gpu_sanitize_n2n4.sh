#!/bin/bash
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_n2n4.py > gpurun_out/sanitize_n2n4_${tool}.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|status|done" gpurun_out/sanitize_n2n4_${tool}.txt | tail -4
done
