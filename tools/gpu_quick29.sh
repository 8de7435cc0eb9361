#!/bin/bash
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 300 python bench.py --steps 3 --warmup 1 --replicas 1 --batch 1 --no-e2e --no-cpu-baseline --candidates 0 --stages > gpurun_out/o_single.json 2> gpurun_out/o_single.err
timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 6 > gpurun_out/o_tp.json 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 6 > gpurun_out/o_tp2.json 2>/dev/null
