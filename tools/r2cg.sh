#!/bin/bash
# optimistic on-chip placement meta: placement tests + configs + wide stages
T=${1:-r2cg}
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 1200 python -u -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_batch.py -m gpu -q --timeout 600 -p no:cacheprovider -x -k "placement or config or batch or pipeline" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
B="--steps 2 --warmup 2 --replicas 1 --batch 1 --no-cpu-baseline --candidates 0 --no-e2e --stages --no-wide-levels"
DP_DEBUG_PLACE=1 timeout 600 python bench.py --variant wide $B > gpurun_out/${T}_wide.json 2> gpurun_out/${T}_wide.err
DP_DEBUG_PLACE=1 DP_PLACE_NO_OPTIMISTIC=1 timeout 600 python bench.py --variant wide $B > gpurun_out/${T}_wide_glob.json 2> gpurun_out/${T}_wide_glob.err
