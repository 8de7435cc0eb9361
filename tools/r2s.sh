#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2s}
for r in 1 4 16; do
DP_DEBUG_SYNC=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --candidates 0 --no-e2e --replicas $r > gpurun_out/${T}_r$r.json 2> gpurun_out/${T}_r$r.err
done
