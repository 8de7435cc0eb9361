#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2ae}
DP_DEBUG_DP=1 timeout 300 python tools/perf_stages.py deep > gpurun_out/${T}_stages_deep.txt 2>&1
PYTHONUNBUFFERED=1 timeout 1200 python -u -m pytest tests/test_gpu_fixpoint.py tests/test_gpu_paths.py tests/test_gpu_configs.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
