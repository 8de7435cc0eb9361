#!/bin/bash
# gate-mode dataflow levels: tests + probe + wide stages
T=${1:-r2bo}
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests/test_gpu_paths.py -m gpu -q --timeout 300 -p no:cacheprovider -x -k "levels" > gpurun_out/${T}_pytest_levels.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_levels.log
timeout 600 python tools/levels_probe.py 7 > gpurun_out/${T}_levels_probe.txt 2>&1; echo "probe rc=$?" >> gpurun_out/${T}_levels_probe.txt
timeout 600 python bench.py --variant wide --steps 2 --warmup 1 --replicas 8 --no-cpu-baseline --candidates 0 --stages --no-e2e > gpurun_out/${T}_wide.json 2> gpurun_out/${T}_wide.err
rm -f gpurun_out/${T}_lv.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_levels_flow_batch' -c 2 \
  -o gpurun_out/${T}_lv python tools/levels_probe.py 1 env > gpurun_out/${T}_ncu.log 2>&1
