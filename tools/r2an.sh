#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2an}
PYTHONUNBUFFERED=1 timeout 1500 python -u -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
DP_DEBUG_SYNC=1 timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --candidates 0 --stages-under-load > gpurun_out/${T}_deep.json 2> gpurun_out/${T}_deep.err
