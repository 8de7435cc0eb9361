#!/bin/bash
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests -m gpu -x -q --timeout 180 -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
bash tools/gpu_place_dbg.sh
