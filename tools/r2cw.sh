#!/bin/bash
# coarse sweep: lane-0 path for nodes with at most 4 in-tile sources; tests + stages
T=${1:-r2cw}
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 700 python -u -m pytest tests/test_gpu_paths.py tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_batch.py -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
B="--steps 2 --warmup 2 --replicas 1 --batch 1 --no-cpu-baseline --candidates 0 --no-e2e --stages --no-wide-levels"
for v in deep wide; do
  timeout 300 python bench.py --variant $v $B > gpurun_out/${T}_${v}.json 2> gpurun_out/${T}_${v}.err
done
