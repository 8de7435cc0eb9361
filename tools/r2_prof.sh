#!/bin/bash
# ncu evidence for the current build: launch list of one single-graph generation and a
# --set full capture of each dominant kernel (one ncu pass per kernel, first launch only),
# summaries via tools/summarize_profiles.py.
D=gpurun_out/prof_${1:-r2}
rm -rf $D; mkdir -p $D
B="--steps 1 --warmup 0 --replicas 1 --batch 1 --no-e2e --no-cpu-baseline --candidates 0 --no-wide-levels"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $D/launches.csv \
  python bench.py --steps 1 --warmup 1 --replicas 1 --batch 1 --no-e2e --no-cpu-baseline --candidates 0 --no-wide-levels > $D/launch.log 2>&1
for k in k_dp_only k_treepeel k_place k_peel2 k_levels_seq k_levels_flow_batch k_rs_scatter; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
    -o $D/prof_$k python bench.py $B > $D/full_$k.log 2>&1
done
DP_DEBUG_SYNC=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --candidates 0 --no-e2e --stages-under-load > $D/under_load.json 2> $D/under_load.err
