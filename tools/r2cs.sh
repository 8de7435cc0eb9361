#!/bin/bash
# throughput A/B on one box: 32 x 4 vs 32 x 6 graphs (e2e at 4 graphs per call in both), twice
T=${1:-r2cs}
mkdir -p gpurun_out
B="--steps 5 --warmup 3 --no-cpu-baseline --candidates 0 --no-wide-levels --e2e-batch 4"
for i in 1 2; do
  timeout 900 python bench.py $B --batch 4 > gpurun_out/${T}_b4_$i.json 2> gpurun_out/${T}_b4_$i.err
  timeout 900 python bench.py $B --batch 6 > gpurun_out/${T}_b6_$i.json 2> gpurun_out/${T}_b6_$i.err
done
