#!/bin/bash
# v6 peel check: parity suite, single-graph stage timings, ncu source profile of k_peel_dp
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
DP_DEBUG_DP=1 timeout 300 python bench.py --steps 2 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 --stages > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
DP_PEEL_V5=1 DP_DEBUG_DP=1 timeout 300 python bench.py --steps 2 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 --stages > gpurun_out/q_bench_v5.json 2> gpurun_out/q_bench_v5.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_peel_dp' -s 1 -c 1 \
  -o gpurun_out/prof_v6 python bench.py --steps 1 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 > gpurun_out/ncu_v6.log 2>&1
