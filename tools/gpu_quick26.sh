#!/bin/bash
mkdir -p gpurun_out
for RK in "32 4" "30 4" "28 4" "32 4"; do set -- $RK
  timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 8 --replicas $1 --batch $2 > gpurun_out/l_r$1_k$2_$RANDOM.json 2>/dev/null
done
