#!/bin/bash
# coarse-graph sweep rework: GPU tests (full suite) + wide / deep stage times
T=${1:-r2bw}
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 1500 python -u -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
B="--steps 2 --warmup 2 --replicas 1 --batch 1 --no-cpu-baseline --candidates 0 --no-e2e --stages --no-wide-levels"
timeout 600 python bench.py --variant wide $B > gpurun_out/${T}_wide.json 2> gpurun_out/${T}_wide.err
timeout 600 python bench.py --variant deep $B > gpurun_out/${T}_deep.json 2> gpurun_out/${T}_deep.err
