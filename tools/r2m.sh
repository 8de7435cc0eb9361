#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2m}
DP_DEBUG_DP=1 timeout 300 python tools/perf_stages.py deep > gpurun_out/${T}_stages_deep.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dp_only -c 1 \
  -o gpurun_out/${T}_prof_dp python tools/prof_dp.py deep > gpurun_out/${T}_ncu_dp.log 2>&1
