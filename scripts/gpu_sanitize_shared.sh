for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_shared.py > gpurun_out/sanitize_shared_${tool}.txt 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_shared_${tool}.txt
done
