#!/bin/bash
mkdir -p gpurun_out
for E in DP_X=1 DP_PEEL_NO_PREFETCH=1; do
  env $E timeout 300 python bench.py --steps 3 --warmup 1 --replicas 1 --batch 1 --no-e2e --no-cpu-baseline --candidates 0 --stages 2>&1 >/dev/null | grep -E "peel" | sed "s/^/$E single /" >> gpurun_out/k.log
  env $E timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 4 > gpurun_out/k_$E.json 2>/dev/null
done
