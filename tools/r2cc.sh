#!/bin/bash
# cluster tree peel: fixpoint tests, stage times per cluster size (deep / wide)
T=${1:-r2cc}
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests/test_gpu_fixpoint.py -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/${T}_pytest_fix.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_fix.log
B="--steps 2 --warmup 2 --replicas 1 --batch 1 --no-cpu-baseline --candidates 0 --no-e2e --stages --no-wide-levels"
for c in def; do
  for v in deep wide; do
    env DP_DEBUG_FIXPOINT=1 $( [ $c = def ] || echo DP_TREE_CLUSTER=$c ) timeout 600 python bench.py --variant $v $B > gpurun_out/${T}_${v}_c$c.json 2> gpurun_out/${T}_${v}_c$c.err
  done
done
