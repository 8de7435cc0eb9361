#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2r}
DP_DEBUG_SYNC=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --candidates 0 --no-e2e > gpurun_out/${T}_deep.json 2> gpurun_out/${T}_deep.err
