#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 3 --replicas 32 --batch 4 --stages-under-load > gpurun_out/e_r32_k4.json 2> gpurun_out/e_r32_k4.err
DP_LEVELS_KAHN=1 timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 3 --replicas 32 --batch 4 --stages-under-load > gpurun_out/e_r32_k4_kahn.json 2> gpurun_out/e_r32_k4_kahn.err
DP_FLOW_AHEAD=32 timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 3 --replicas 32 --batch 4 --stages-under-load > gpurun_out/e_r32_k4_a32.json 2> gpurun_out/e_r32_k4_a32.err
