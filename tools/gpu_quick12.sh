#!/bin/bash
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 600 python -u -m pytest tests/test_gpu_paths.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/q_paths.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_paths.log
for A in auto 16 64 256 1024; do
  if [ $A = auto ]; then unset DP_FLOW_AHEAD; else export DP_FLOW_AHEAD=$A; fi
  echo "== ahead $A" >> gpurun_out/q_flow.log
  timeout 300 python bench.py --steps 2 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 --stages 2>&1 >/dev/null | grep -E "levels|generate" >> gpurun_out/q_flow.log
  timeout 300 python bench.py --variant wide --steps 2 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 --stages 2>&1 >/dev/null | grep -E "levels|generate" | sed 's/^/wide /' >> gpurun_out/q_flow.log
done
