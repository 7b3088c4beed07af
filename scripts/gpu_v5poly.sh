for v in "" p4 p6 p8; do echo "== $v"; PA_LIB_VARIANT=$v PA_PREFILL=5 timeout 300 python scripts/prefill_bench.py --no-cpu-baseline --configs p_2k,p_sharegpt,p_chunk256 2>&1 | cut -c1-120; done
PA_LIB_VARIANT=p6 PA_PREFILL=5 timeout 600 python -m pytest tests/test_gpu_prefill.py -q -x 2>&1 | tail -2
