#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b2.json 2> gpurun_out/b2.err
timeout 600 python bench.py --no-cpu-baseline --candidates 0 > gpurun_out/b3.json 2> gpurun_out/b3.err
