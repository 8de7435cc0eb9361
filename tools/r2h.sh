#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2h}
DP_DEBUG_DP=1 timeout 300 python tools/perf_stages.py deep > gpurun_out/${T}_stages_deep.txt 2>&1
