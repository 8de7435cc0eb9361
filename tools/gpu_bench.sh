#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 300 python bench.py --steps 3 --warmup 3 --replicas 16 --no-cpu-baseline --candidates 0 > gpurun_out/bench_r16.json 2> gpurun_out/bench_r16.err
