#!/bin/bash
# A/B of the bulk L2 row prefetch in the dataflow level kernel (separate processes, alternating)
T=${1:-r2bu}
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests/test_gpu_paths.py -m gpu -q --timeout 300 -p no:cacheprovider -x -k "levels" > gpurun_out/${T}_pytest_levels.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_levels.log
for i in 1 2 3; do
  echo "== prefetch $i"; python tools/levels_probe.py 7 env
  echo "== no-prefetch $i"; DP_FLOW_NO_PREFETCH=1 python tools/levels_probe.py 7 env
done > gpurun_out/${T}_ab.txt 2>&1
