#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_peel_dp' -s 1 -c 1 \
  -o gpurun_out/prof_peel python bench.py --steps 1 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 > gpurun_out/ncu_peel.log 2>&1
