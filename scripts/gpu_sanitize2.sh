for sched in coop grid pcoop persistent; do
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 5 python scripts/sanitize.py $sched > gpurun_out/racecheck_${sched}.txt 2>&1
  echo "$sched: $(grep -E 'SUMMARY' gpurun_out/racecheck_${sched}.txt)"
done
