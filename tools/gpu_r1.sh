#!/bin/bash
# One GPU session: parity suite, smoke, bench, ncu launch list + full capture of the top kernels.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --stages > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 > gpurun_out/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_kahn_fwd|k_kahn_bwd|k_peel_dp' -s 6 -c 4 \
  -o gpurun_out/prof_r1 python bench.py --steps 1 --warmup 1 --replicas 1 --no-e2e --no-cpu-baseline --candidates 0 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
