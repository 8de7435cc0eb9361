#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_probe.py (round-2 kernels)
T=${1:-r2cl}
mkdir -p gpurun_out
timeout 300 python tools/sanitize_probe.py > gpurun_out/${T}_probe_plain.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_probe_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_probe.py > gpurun_out/${T}_san_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${T}_san_${tool}.log
done
