#!/bin/bash
# throughput mode: streams x graphs-per-call sweep on the current build
T=${1:-r2cj}
mkdir -p gpurun_out
B="--steps 3 --warmup 3 --no-cpu-baseline --candidates 0 --no-e2e --no-wide-levels"
for rk in "32 4" "32 6" "24 8" "16 8" "32 8"; do
  set -- $rk
  timeout 900 python bench.py $B --replicas $1 --batch $2 > gpurun_out/${T}_r$1_b$2.json 2> gpurun_out/${T}_r$1_b$2.err
done
