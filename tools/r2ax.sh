#!/bin/bash
# placement ncu captures (wide + deep coarse graphs) and the new batch error-order test
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -m gpu -q -p no:cacheprovider > gpurun_out/r2ax_batch.log 2>&1; echo "rc=$?" >> gpurun_out/r2ax_batch.log
for v in wide deep; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_place -c 1 -f -o gpurun_out/r2ax_place_$v python tools/prof_place.py $v > gpurun_out/r2ax_ncu_$v.log 2>&1
done
