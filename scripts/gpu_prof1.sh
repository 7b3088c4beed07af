CFG=${1:-c2_alpaca}
K=${2:-paged_attention_persistent_kernel}
TAG=${3:-x}
ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
    -o gpurun_out/prof_${CFG}_${TAG} -f \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_${CFG}_${TAG}.log 2>&1
