#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --candidates 0 --steps 5 --e2e-steps 5 --warmup 3 --stages > gpurun_out/j1.json 2> gpurun_out/j1.err
DP_PIN_GROW=1 timeout 600 python bench.py --no-cpu-baseline --candidates 0 --steps 5 --e2e-steps 5 --warmup 3 --stages > gpurun_out/j2.json 2> gpurun_out/j2.err
