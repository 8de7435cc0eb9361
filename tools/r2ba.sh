#!/bin/bash
# throughput structure: stages under load, replica/batch sweep, coarse levels kernel choice
T=${1:-r2ba}
mkdir -p gpurun_out
B="--steps 3 --warmup 3 --no-cpu-baseline --candidates 0 --no-e2e"
timeout 600 python bench.py $B --stages-under-load > gpurun_out/${T}_load.json 2> gpurun_out/${T}_load.err
for rk in "16 8" "24 8" "32 6" "32 8" "48 4"; do
  set -- $rk
  timeout 600 python bench.py $B --replicas $1 --batch $2 > gpurun_out/${T}_r$1_b$2.json 2> gpurun_out/${T}_r$1_b$2.err
done
for v in deep wide; do
  DP_COARSE_FLOW=1 timeout 600 python bench.py --variant $v --steps 2 --warmup 3 --replicas 1 --batch 1 --no-cpu-baseline --candidates 0 --no-e2e --stages --no-check > gpurun_out/${T}_flow_$v.json 2> gpurun_out/${T}_flow_$v.err
done
