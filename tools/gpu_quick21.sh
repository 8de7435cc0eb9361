#!/bin/bash
mkdir -p gpurun_out
DP_DEBUG_PIPE=1 timeout 600 python bench.py --no-cpu-baseline --candidates 0 --steps 1 --warmup 3 > gpurun_out/g_e2e.json 2> gpurun_out/g_e2e.err
timeout 600 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --candidates 8192 --no-e2e > gpurun_out/g_cand.json 2> gpurun_out/g_cand.err
