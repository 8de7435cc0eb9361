#!/bin/bash
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests/test_gpu_configs.py -x -q --timeout 600 -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
