#!/bin/bash
mkdir -p gpurun_out
DP_DEBUG_PLACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 > /dev/null 2> gpurun_out/q_place_dbg.err
DP_DEBUG_PLACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --replicas 1 --variant wide --no-e2e --no-cpu-baseline --candidates 0 > /dev/null 2>> gpurun_out/q_place_dbg.err
