#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --steps 3 --warmup 2 --replicas 32 --no-e2e --no-cpu-baseline --candidates 0 --stages-under-load > gpurun_out/q_load.json 2> gpurun_out/q_load.err
DP_SPIN_SYNC=1 timeout 300 python bench.py --steps 3 --warmup 2 --replicas 32 --no-e2e --no-cpu-baseline --candidates 0 > gpurun_out/q_load_spin.json 2> gpurun_out/q_load_spin.err
timeout 300 python bench.py --steps 3 --warmup 2 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 > gpurun_out/q_load_r1.json 2> gpurun_out/q_load_r1.err
