#!/bin/bash
# coarse CPD peel: v6 dense mode on the coarse graphs vs the v5 peel
T=${1:-r2by}
mkdir -p gpurun_out
B="--steps 2 --warmup 2 --replicas 1 --batch 1 --no-cpu-baseline --candidates 0 --no-e2e --stages --no-wide-levels"
for v in wide deep; do
  timeout 600 python bench.py --variant $v $B > gpurun_out/${T}_${v}_v6.json 2> gpurun_out/${T}_${v}_v6.err
  DP_PEEL_V6_DENSE=0 timeout 600 python bench.py --variant $v $B > gpurun_out/${T}_${v}_v5.json 2> gpurun_out/${T}_${v}_v5.err
done
