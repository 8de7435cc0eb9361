#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2f}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_dp_only|k_treepeel' -c 2 \
  -o gpurun_out/${T}_prof_dp python tools/prof_dp.py deep > gpurun_out/${T}_ncu_dp.log 2>&1
