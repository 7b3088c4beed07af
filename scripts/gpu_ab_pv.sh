# FHFMA P.V (default) vs fp32-weight P.V (libpagedattn_base.so, -DPA_PV_F32): tests + A/B
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_pv.txt; cat gpurun_out/pytest_pv.txt
V=base CFGS="c5_beam c3_fork c3_parallel c2_alpaca c2_sharegpt c4_sharegpt" bash scripts/gpu_ab.sh > gpurun_out/ab_pv.txt 2>&1; cat gpurun_out/ab_pv.txt
