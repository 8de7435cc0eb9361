#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 300 python bench.py --steps 2 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 --stages > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
timeout 300 python bench.py --steps 2 --warmup 1 --replicas 1 --variant wide --no-e2e --no-cpu-baseline --candidates 0 --stages > gpurun_out/q_wide.json 2> gpurun_out/q_wide.err
