# N1 shared decode as C5's default: GPU tests, bench lines (shared vs coop), ncu captures
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_gpu_r01.txt; cat gpurun_out/pytest_gpu_r01.txt
for rep in 1 2; do
  timeout 300 python bench.py --config c5_beam --steps 500 --warmup 10 --no-cpu-baseline --no-e2e 2>>gpurun_out/sh.err > gpurun_out/c5_shared_$rep.json
  timeout 300 python bench.py --config c5_beam --steps 500 --warmup 10 --no-cpu-baseline --no-e2e --shared 0 2>>gpurun_out/sh.err > gpurun_out/c5_coop_$rep.json
  for f in gpurun_out/c5_shared_$rep.json gpurun_out/c5_coop_$rep.json; do
    python -c "import json,sys; d=json.load(open('$f')); print('$f', d['config']['decode_kernel'], round(d['us_per_step'],1), round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['gpu_launches'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
bash scripts/gpu_profile.sh c5_beam r01 > /dev/null 2>&1
ls gpurun_out/*c5_beam*
