#!/bin/bash
# Round-2 evidence after the level-pass rework: GPU tests, smoke, bench line (with the wide
# level-pass roofline), wide variant stages, ncu --set full of k_levels_flow_batch (wide + deep).
T=${1:-r2bt}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/${T}_smi.csv
PYTHONUNBUFFERED=1 timeout 1500 python -u -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 1200 python bench.py --stages > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?" >> gpurun_out/${T}_bench.err
timeout 600 python bench.py --variant wide --steps 2 --warmup 1 --replicas 8 --no-cpu-baseline --candidates 0 --stages > gpurun_out/${T}_wide.json 2> gpurun_out/${T}_wide.err
rm -f gpurun_out/${T}_lv.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_levels_flow_batch' -c 2 \
  -o gpurun_out/${T}_lv python tools/levels_probe.py 1 env > gpurun_out/${T}_ncu.log 2>&1
