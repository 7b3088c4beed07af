# ncu evidence for the dominant kernel (run under gpurun, 1 GPU).
#   launches.csv : every libpagedattn launch of a short bench run (cold-cache, serialised)
#   prof_attn    : one --set full capture of paged_attention_kernel (+ source view)
CFG=${1:-c2_sharegpt}
TAG=${2:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'paged_attention|reshape_and_cache|copy_blocks' --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv \
    python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_${CFG}_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:paged_attention -s 3 -c 1 \
    -o gpurun_out/prof_attn_${CFG}_${TAG} -f \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_${CFG}_${TAG}.log 2>&1
ls -la gpurun_out
