#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2v}
DP_DEBUG_PLACE=1 timeout 300 python tools/prof_place.py deep > gpurun_out/${T}_place.txt 2>&1
DP_DEBUG_PLACE=1 timeout 300 python tools/prof_place.py wide > gpurun_out/${T}_place_wide.txt 2>&1
