#!/bin/bash
# tree peel: targeted GPU tests, wide/deep stage timings, then the whole GPU suite
mkdir -p gpurun_out
T=${1:-r2c}
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests/test_gpu_fixpoint.py tests/test_gpu_paths.py tests/test_gpu_switches.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/${T}_pytest_fix.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_fix.log
DP_DEBUG_DP=1 DP_DEBUG_FIXPOINT=1 timeout 300 python tools/perf_stages.py wide > gpurun_out/${T}_stages_wide.txt 2>&1
DP_DEBUG_DP=1 DP_DEBUG_FIXPOINT=1 timeout 300 python tools/perf_stages.py deep > gpurun_out/${T}_stages_deep.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --candidates 0 --no-e2e --stages > gpurun_out/${T}_deep.json 2> gpurun_out/${T}_deep.err
timeout 600 python bench.py --variant wide --steps 2 --warmup 1 --replicas 8 --no-cpu-baseline --candidates 0 --no-e2e --stages > gpurun_out/${T}_wide.json 2> gpurun_out/${T}_wide.err
PYTHONUNBUFFERED=1 timeout 1500 python -u -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
