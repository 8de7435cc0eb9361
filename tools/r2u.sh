#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2u}
DP_DEBUG_PLACE=1 timeout 300 python tools/prof_place.py deep > gpurun_out/${T}_place.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_place -c 1 \
  -o gpurun_out/${T}_prof_place python tools/prof_place.py deep > gpurun_out/${T}_ncu_place.log 2>&1
