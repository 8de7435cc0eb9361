#!/bin/bash
# coarse graphs through the tree peel (DP_COARSE_TREE) vs the one-warp peel
T=${1:-r2cp}
mkdir -p gpurun_out
B="--steps 2 --warmup 2 --replicas 1 --batch 1 --no-cpu-baseline --candidates 0 --no-e2e --stages --no-wide-levels"
for v in deep wide; do
  DP_DEBUG_FIXPOINT=1 DP_COARSE_TREE=1 timeout 600 python bench.py --variant $v $B > gpurun_out/${T}_${v}_tree.json 2> gpurun_out/${T}_${v}_tree.err
  DP_DEBUG_FIXPOINT=1 DP_COARSE_TREE=1 DP_PEEL_FIXPOINT=1 timeout 600 python bench.py --variant $v $B > gpurun_out/${T}_${v}_treeforce.json 2> gpurun_out/${T}_${v}_treeforce.err
done
