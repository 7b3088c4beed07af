for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_${tool}.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_${tool}.txt
done
