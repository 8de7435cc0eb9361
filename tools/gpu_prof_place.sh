#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --steps 1 --warmup 1 --replicas 1 --variant wide --no-e2e --no-cpu-baseline --candidates 0 --stages > gpurun_out/q_wide.json 2> gpurun_out/q_wide.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_place' -s 1 -c 1 \
  -o gpurun_out/prof_place python bench.py --steps 1 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 > gpurun_out/ncu_place.log 2>&1
