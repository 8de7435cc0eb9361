#!/bin/bash
mkdir -p gpurun_out
for RK in "16 8" "24 5" "32 4" "16 8"; do set -- $RK
  timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 5 --replicas $1 --batch $2 > gpurun_out/v_tmp.json 2>/dev/null
  echo "$RK $(python -c "import json;d=json.load(open('gpurun_out/v_tmp.json'));print(round(d['value']/1e6,1), d['step_ms_all'])")" >> gpurun_out/v.log
done
