#!/bin/bash
mkdir -p gpurun_out
for RK in "16 8" "32 4"; do set -- $RK
  timeout 600 python bench.py --no-cpu-baseline --candidates 0 --steps 5 --e2e-steps 4 --replicas $1 --batch $2 > gpurun_out/w_tmp.json 2>/dev/null
  echo "$RK $(python -c "import json;d=json.load(open('gpurun_out/w_tmp.json'));print(round(d['value']/1e6,1), d['step_ms_all'], round(d['e2e']['value']/1e6,1), d['e2e']['ms_per_step'])")" >> gpurun_out/w.log
done
