#!/bin/bash
mkdir -p gpurun_out
DP_PEEL_LATE_ROWS=1 PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests/test_gpu_paths.py tests/test_gpu_batch.py tests/test_gpu_configs.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
for E in DP_X=1 DP_PEEL_LATE_ROWS=1 DP_X=1 DP_PEEL_LATE_ROWS=1; do
  env $E timeout 300 python bench.py --steps 3 --warmup 1 --replicas 1 --batch 1 --no-e2e --no-cpu-baseline --candidates 0 --stages 2>&1 >/dev/null | grep -E "peel\+dp|cpd" | sed "s/^/$E /" >> gpurun_out/r.log
done
DP_PEEL_LATE_ROWS=1 timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 6 > gpurun_out/r_tp.json 2>/dev/null
