timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_r01.txt; tail -1 gpurun_out/pytest_gpu_r01.txt
for rep in 1 2; do
  timeout 300 python bench.py --config c5_beam --steps 500 --warmup 10 --no-cpu-baseline --no-e2e 2>>gpurun_out/sh.err > gpurun_out/c5_shared_$rep.json
  python -c "import json,sys; d=json.load(open('gpurun_out/c5_shared_$rep.json')); print(d['config']['decode_kernel'], round(d['us_per_step'],1), round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
SWEEP_SHAPES="coop,4,2,1;shared4,2,3,1;shared4,2,2,1" timeout 300 python scripts/sweep.py c5_beam 2>&1 | grep -v Warn
bash scripts/gpu_profile.sh c5_beam r01 > /dev/null 2>&1
