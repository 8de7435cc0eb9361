#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "simulate or candidates or bruteforce or config" > gpurun_out/q_pytest_sim.log 2>&1; echo "rc=$?" >> gpurun_out/q_pytest_sim.log
timeout 300 python bench.py --steps 2 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 16384 > gpurun_out/q_cand.json 2> gpurun_out/q_cand.err
