#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_estimation.py tests/test_gpu_paths.py -x -q > gpurun_out/q_pytest_est.log 2>&1; echo "rc=$?" >> gpurun_out/q_pytest_est.log
