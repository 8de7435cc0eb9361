#!/bin/bash
mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/q_flow2.log
  env "$@" timeout 300 python bench.py --steps 2 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 --stages 2>&1 >/dev/null | grep -E "levels|generate" >> gpurun_out/q_flow2.log
  env "$@" timeout 300 python bench.py --variant wide --steps 2 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 --stages 2>&1 >/dev/null | grep -E "levels|generate" | sed 's/^/wide /' >> gpurun_out/q_flow2.log
}
run DP_X=0
run DP_FLOW_SLEEP=0
run DP_FLOW_SLEEP=64
run DP_FLOW_SLEEP=128
run DP_FLOW_SLEEP=1024
run DP_LEVELS_FLOW=1
run DP_LEVELS_FLOW=1 DP_FLOW_SLEEP=0
