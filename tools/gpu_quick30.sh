#!/bin/bash
mkdir -p gpurun_out
DP_PEEL_EXCLUSIVE=1 PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests/test_gpu_batch.py tests/test_gpu_paths.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
for E in DP_X=1 DP_PEEL_EXCLUSIVE=1 DP_X=1 DP_PEEL_EXCLUSIVE=1; do
  env $E timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 6 > gpurun_out/p_$E_$RANDOM.json 2>/dev/null
  echo "$E $(python -c "import json,glob,os;f=max(glob.glob('gpurun_out/p_*.json'),key=os.path.getmtime);d=json.load(open(f));print(d['value']/1e6, d['step_ms_all'])")" >> gpurun_out/p.log
done
