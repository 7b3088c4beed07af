CFG=${1:-c2_alpaca}
for sched in persistent grid; do
PA_SCHED=$sched ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'paged_attention|reshape_and_cache|copy_blocks|build_worklist' --csv --log-file gpurun_out/launches_${CFG}_${sched}.csv \
    python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
