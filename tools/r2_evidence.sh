#!/bin/bash
# Round-2 evidence on the current build: GPU tests, smoke, the default bench line, the
# reference arm, and the drop-in timing.  Outputs under gpurun_out/ (tag = $1).
T=${1:-r2a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/${T}_smi.csv
lscpu > gpurun_out/${T}_lscpu.txt
PYTHONUNBUFFERED=1 timeout 1500 python -u -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?" >> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "ref rc=$?" >> gpurun_out/${T}_bench_ref.err
timeout 600 python bench.py --variant wide --steps 2 --warmup 1 --replicas 8 --no-cpu-baseline --candidates 0 --stages > gpurun_out/${T}_wide.json 2> gpurun_out/${T}_wide.err
