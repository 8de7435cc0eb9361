#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 1 --replicas 32 --no-e2e --no-cpu-baseline --candidates 0 --stages-under-load > gpurun_out/q_load.json 2> gpurun_out/q_load.err
