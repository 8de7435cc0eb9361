#!/bin/bash
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests/test_gpu_configs.py tests/test_gpu_paths.py tests/test_gpu_batch.py -x -q --timeout 600 -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 300 python bench.py --variant wide --steps 2 --warmup 1 --replicas 1 --batch 1 --no-e2e --no-cpu-baseline --candidates 0 --stages 2>&1 >/dev/null | grep -E "generate|levels" > gpurun_out/x.log
timeout 300 python bench.py --steps 2 --warmup 1 --replicas 1 --batch 1 --no-e2e --no-cpu-baseline --candidates 0 --stages 2>&1 >/dev/null | grep -E "generate|levels" >> gpurun_out/x.log
