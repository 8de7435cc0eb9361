#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
DP_DEBUG_DP=1 timeout 300 python bench.py --steps 2 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 --stages > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
rm -f gpurun_out/exp_replicas.txt
for R in 1 8 16 32 48; do
  timeout 300 python bench.py --steps 2 --warmup 1 --replicas $R --no-cpu-baseline --candidates 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print($R, d['ms_per_step'], d['value']/1e6, d['single_graph']['ms'], d['e2e']['value']/1e6, d['e2e']['ms_per_step'])" >> gpurun_out/exp_replicas.txt
done
