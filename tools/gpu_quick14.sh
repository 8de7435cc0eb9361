#!/bin/bash
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 400 python bench.py --no-cpu-baseline --candidates 0 > gpurun_out/b6.json 2> gpurun_out/b6.err
for R in 48 64; do timeout 400 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --replicas $R > gpurun_out/b_r$R.json 2> gpurun_out/b_r$R.err; done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/b_r64.err
