#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 2 --stages-under-load > gpurun_out/s_tp.json 2> gpurun_out/s_tp.err
