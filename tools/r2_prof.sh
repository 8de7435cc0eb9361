#!/bin/bash
# ncu evidence for the current build: launch list of one single-graph generation and a
# --set full capture of the dominant kernels (summaries via tools/summarize_profiles.py).
D=gpurun_out/prof_${1:-r2}
rm -rf $D; mkdir -p $D
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $D/launches.csv \
  python bench.py --steps 1 --warmup 1 --replicas 1 --batch 1 --no-e2e --no-cpu-baseline --candidates 0 --no-wide-levels > $D/launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:'k_dp_only|k_treepeel|k_levels_flow_batch|k_place|k_levels_seq|k_peel2|k_rs_scatter' -c 8 \
  -o $D/prof_main python bench.py --steps 1 --warmup 0 --replicas 1 --batch 1 --no-e2e --no-cpu-baseline --candidates 0 --no-wide-levels > $D/full.log 2>&1
DP_DEBUG_SYNC=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --candidates 0 --no-e2e --stages-under-load > $D/under_load.json 2> $D/under_load.err
