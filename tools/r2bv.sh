#!/bin/bash
# wide variant secondary stages under alternative kernel choices (coarse levels / coarse peel)
T=${1:-r2bv}
mkdir -p gpurun_out
B="--variant wide --steps 2 --warmup 2 --replicas 1 --batch 1 --no-cpu-baseline --candidates 0 --no-e2e --stages --no-wide-levels"
for mode in default flow fixpoint flowfix; do
  case $mode in
    default) E="";;
    flow) E="DP_COARSE_FLOW=1";;
    fixpoint) E="DP_PEEL_FIXPOINT=1";;
    flowfix) E="DP_COARSE_FLOW=1 DP_PEEL_FIXPOINT=1";;
  esac
  env $E DP_DEBUG_FIXPOINT=1 timeout 600 python bench.py $B > gpurun_out/${T}_$mode.json 2> gpurun_out/${T}_$mode.err
done
