#!/bin/bash
# DP v5 dead-row skip: fixpoint/paths/configs tests + deep/wide stages with and without
T=${1:-r2co}
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 1500 python -u -m pytest tests/test_gpu_fixpoint.py tests/test_gpu_paths.py tests/test_gpu_configs.py tests/test_gpu_batch.py -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
B="--steps 3 --warmup 2 --replicas 1 --batch 1 --no-cpu-baseline --candidates 0 --no-e2e --stages --no-wide-levels"
for v in deep wide; do
  timeout 600 python bench.py --variant $v $B > gpurun_out/${T}_${v}.json 2> gpurun_out/${T}_${v}.err
  DP_DP5_NO_SKIP=1 timeout 600 python bench.py --variant $v $B > gpurun_out/${T}_${v}_noskip.json 2> gpurun_out/${T}_${v}_noskip.err
done
