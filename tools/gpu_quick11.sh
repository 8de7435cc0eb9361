#!/bin/bash
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 400 python bench.py --no-cpu-baseline --candidates 0 --stages > gpurun_out/b4.json 2> gpurun_out/b4.err
timeout 400 python bench.py --no-cpu-baseline --candidates 0 > gpurun_out/b5.json 2> gpurun_out/b5.err
