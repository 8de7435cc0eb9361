#!/bin/bash
# placement v3 check: placement-heavy GPU tests, phase timings (deep, wide), stage timings
T=${1:-r2ay}
mkdir -p gpurun_out
for v in deep wide; do
  DP_DEBUG_PLACE=1 timeout 300 python tools/prof_place.py $v > gpurun_out/${T}_place_$v.txt 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_devices.py tests/test_gpu_batch.py tests/test_gpu_configs.py tests/test_gpu_resident.py tests/test_gpu_switches.py -m gpu -q -x -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --candidates 0 --stages > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
for v in deep wide; do timeout 300 python tools/prof_tree.py $v > gpurun_out/${T}_tree_$v.txt 2>&1; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --candidates 0 --lockstep > gpurun_out/${T}_bench_lock.json 2> gpurun_out/${T}_bench_lock.err
