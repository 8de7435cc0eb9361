#!/bin/bash
mkdir -p gpurun_out
DP_DEBUG_PIPE=1 timeout 600 python bench.py --no-cpu-baseline --candidates 0 --steps 1 --warmup 3 > gpurun_out/i_e2e.json 2> gpurun_out/i_e2e.err
timeout 600 python bench.py --no-cpu-baseline --candidates 0 --steps 3 --warmup 3 > gpurun_out/i2_e2e.json 2> gpurun_out/i2_e2e.err
