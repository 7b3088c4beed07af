#!/bin/bash
# Round-2 evidence: ncu launch list of the default bench command, one --set full capture of
# the dominant kernel per config (rotated caches, plan), summarised by scripts/ncu_summary.py
mkdir -p gpurun_out/r02prof
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 40 --csv --log-file gpurun_out/r02prof/launches_c2_sharegpt.csv \
    python bench.py --steps 20 --warmup 10 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/r02prof/launches_c2_sharegpt.log 2>&1
for spec in "c2_sharegpt:paged_attention_coop" "c2_alpaca:paged_attention_coop" "c4_long:paged_attention_coop" \
            "c3_parallel:paged_attention_coop" "c5_beam:group_tc"; do
  cfg=${spec%%:*}; k=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -o gpurun_out/r02prof/$cfg \
      python bench.py --config $cfg --steps 3 --warmup 8 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/r02prof/$cfg.log 2>&1
done
