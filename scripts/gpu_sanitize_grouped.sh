#!/bin/bash
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_grouped.py > gpurun_out/sanitize_grouped_${tool}.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|done" gpurun_out/sanitize_grouped_${tool}.txt | tail -3
done
