#!/bin/bash
# Round evidence: full bench line, reference arm, ncu launch list and full captures of the
# dominant kernels on the current build (summaries go to profiles/ via summarize_profiles.py).
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/ev_smi.csv
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err
timeout 300 python bench.py --variant wide --steps 2 --warmup 1 --replicas 8 --no-cpu-baseline --candidates 0 --stages > gpurun_out/ev_wide.json 2> gpurun_out/ev_wide.err
rm -f gpurun_out/launches*.csv gpurun_out/*.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 > gpurun_out/ev_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_peel_dp|k_levels_flow|k_place|k_levels_seq' -c 6 \
  -o gpurun_out/prof_main python bench.py --steps 1 --warmup 0 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 > gpurun_out/ev_ncu_full.log 2>&1
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/ev_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev_smoke.log
