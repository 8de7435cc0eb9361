#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2q}
for cfg in "32 4" "16 8" "16 4" "32 4 spin" "16 8 spin"; do
  set -- $cfg
  if [ "$3" = "spin" ]; then export DP_SPIN_SYNC=1; else unset DP_SPIN_SYNC; fi
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --candidates 0 --no-e2e --replicas $1 --batch $2 > gpurun_out/${T}_r$1_b$2_$3.json 2> gpurun_out/${T}_r$1_b$2_$3.err
done
