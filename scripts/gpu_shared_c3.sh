# N1 shared kernel on C3 (parallel sampling): shapes, and one ncu capture on c3_fork
SWEEP_SHAPES="coop,4,2,1;shared6,1,4,1;shared6,1,2,1;shared6,1,3,1;shared6,1,2,2;shared2,4,2,1;shared2,4,4,1;shared3,2,2,1;shared3,2,4,1" \
  timeout 900 python scripts/sweep.py c3_fork c3_parallel 2>&1 | grep -v Warn
ncu --set full --clock-control none -k regex:paged_attention_shared -s 3 -c 1 -o gpurun_out/prof_shared_c3_fork -f \
  python bench.py --config c3_fork --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --shared 6 > gpurun_out/prof_shared_c3.log 2>&1
ncu --set full --clock-control none -k regex:paged_attention_coop -s 3 -c 1 -o gpurun_out/prof_coop_c3_fork -f \
  python bench.py --config c3_fork --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_coop_c3.log 2>&1
ls gpurun_out/*.ncu-rep
