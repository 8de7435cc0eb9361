#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over tools/sanitize_probe.py, an ncu
# full capture of the candidate simulator (k_sim), and the C++ drop-in timed at config #4
# against the reference's own objects.  Outputs under gpurun_out/ (tag = $1).
T=${1:-r2b}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_probe.py > gpurun_out/${T}_san_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${T}_san_${tool}.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_sim' -c 2 \
  -o gpurun_out/${T}_prof_sim python bench.py --steps 3 --warmup 3 --replicas 1 --no-e2e --no-cpu-baseline --no-check --candidates 8192 > gpurun_out/${T}_ncu_sim.log 2>&1
timeout 900 build/dropin_bench_b200 1000000 1024 3 > gpurun_out/${T}_dropin_b200.txt 2>&1
timeout 900 build/dropin_bench_ref 1000000 1024 1 > gpurun_out/${T}_dropin_ref.txt 2>&1
