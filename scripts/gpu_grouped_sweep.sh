# grouped (N1 tensor-core) decode: parity, then (slots per stage, stages) sweep vs coop
timeout 300 python -m pytest tests/test_gpu_grouped.py -q -x 2>&1 | tail -2
PA_GROUP_SLOTS=1 timeout 300 python -m pytest tests/test_gpu_grouped.py -q -x 2>&1 | tail -1
b() { timeout 300 python bench.py --config $1 --grouped $2 --steps 300 --warmup 10 --no-cpu-baseline --no-e2e --no-prefill 2>>gpurun_out/ab.err |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$3', d['config']['workload'], round(d['us_per_step'],1), round(r['achieved']), round(r['frac'],3))"; }
for c in ${CFGS:-c5_beam c3_parallel c3_fork}; do
  b $c 0 coop
  for sc in "1 2" "1 4" "2 2" "2 3" "4 2" "1 6"; do set -- $sc; PA_GROUP_SLOTS=$1 PA_GROUP_STG=$2 b $c -1 "gsl$1,stg$2"; done
done
