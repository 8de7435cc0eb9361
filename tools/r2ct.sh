#!/bin/bash
# in-edge maxima with lanes = devices: placement / config tests + phase times A/B
T=${1:-r2ct}
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 700 python -u -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_devices.py tests/test_gpu_batch.py tests/test_gpu_resident.py -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
B="--steps 2 --warmup 2 --replicas 1 --batch 1 --no-cpu-baseline --candidates 0 --no-e2e --stages --no-wide-levels"
for v in deep wide; do
  DP_DEBUG_PLACE=1 timeout 300 python bench.py --variant $v $B > gpurun_out/${T}_${v}.json 2> gpurun_out/${T}_${v}.err
  DP_DEBUG_PLACE=1 DP_PLACE_INEDGE_OLD=1 timeout 300 python bench.py --variant $v $B > gpurun_out/${T}_${v}_old.json 2> gpurun_out/${T}_${v}_old.err
done
