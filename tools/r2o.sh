#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2o}
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --candidates 0 --no-e2e --stages-under-load > gpurun_out/${T}_deep.json 2> gpurun_out/${T}_deep.err
