#!/bin/bash
# split tree-peel proof: full GPU suite + deep/wide stages (default) + fused A/B
T=${1:-r2cm}
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 1500 python -u -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
B="--steps 2 --warmup 2 --replicas 1 --batch 1 --no-cpu-baseline --candidates 0 --no-e2e --stages --no-wide-levels"
for v in deep wide; do
  DP_DEBUG_FIXPOINT=1 timeout 600 python bench.py --variant $v $B > gpurun_out/${T}_${v}.json 2> gpurun_out/${T}_${v}.err
  DP_DEBUG_FIXPOINT=1 DP_TREE_FUSED_PROOF=1 timeout 600 python bench.py --variant $v $B > gpurun_out/${T}_${v}_fused.json 2> gpurun_out/${T}_${v}_fused.err
done
