#!/bin/bash
mkdir -p gpurun_out
for RK in "32 2" "28 2" "30 2" "32 2" "20 3"; do set -- $RK
  timeout 500 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 8 --replicas $1 --batch $2 --stages-under-load > gpurun_out/c_r$1_k$2.json 2>> gpurun_out/c_r$1_k$2.err
done
