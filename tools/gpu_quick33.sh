#!/bin/bash
mkdir -p gpurun_out
for E in DP_X=1 DP_FLOW_SLEEP=1024 DP_FLOW_AHEAD=64 DP_LEVELS_KAHN=1 "DP_FLOW_AHEAD=64 DP_FLOW_SLEEP=1024"; do
  env $E timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 4 > gpurun_out/t_tmp.json 2>/dev/null
  echo "$E $(python -c "import json;d=json.load(open('gpurun_out/t_tmp.json'));print(round(d['value']/1e6,1), d['step_ms_all'])")" >> gpurun_out/t.log
done
