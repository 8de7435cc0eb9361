#!/bin/bash
mkdir -p gpurun_out
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/b2.json 2> gpurun_out/b2.err
timeout 400 python bench.py --no-cpu-baseline --candidates 0 > gpurun_out/b3.json 2> gpurun_out/b3.err
timeout 600 python -m pytest tests/test_gpu_estimation.py tests/test_gpu_paths.py tests/test_gpu_parity.py -x -q -k "estimation or paths or reference_suite or placement or pipeline" > gpurun_out/q_pytest_est.log 2>&1; echo "rc=$?" >> gpurun_out/q_pytest_est.log
