#!/bin/bash
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 600 python bench.py --no-cpu-baseline --candidates 0 --steps 5 --e2e-steps 5 --warmup 3 --stages > gpurun_out/n1.json 2> gpurun_out/n1.err
