#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2w}
DP_DEBUG_PLACE=1 timeout 300 python tools/prof_place.py deep > gpurun_out/${T}_place.txt 2>&1
DP_DEBUG_PLACE=1 timeout 300 python tools/prof_place.py wide > gpurun_out/${T}_place_wide.txt 2>&1
PYTHONUNBUFFERED=1 timeout 1200 python -u -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_devices.py tests/test_gpu_batch.py tests/test_gpu_switches.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
