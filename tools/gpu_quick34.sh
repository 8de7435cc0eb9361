#!/bin/bash
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests/test_gpu_paths.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 300 python bench.py --steps 3 --warmup 1 --replicas 1 --batch 1 --no-e2e --no-cpu-baseline --candidates 0 --stages 2>&1 >/dev/null | grep -E "generate|levels" > gpurun_out/u.log
timeout 300 python bench.py --variant wide --steps 2 --warmup 1 --replicas 1 --batch 1 --no-e2e --no-cpu-baseline --candidates 0 --stages 2>&1 >/dev/null | grep -E "generate|levels" | sed 's/^/wide /' >> gpurun_out/u.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 5 > gpurun_out/u_tmp.json 2>/dev/null
  echo "tp $(python -c "import json;d=json.load(open('gpurun_out/u_tmp.json'));print(round(d['value']/1e6,1), d['step_ms_all'])")" >> gpurun_out/u.log; done
