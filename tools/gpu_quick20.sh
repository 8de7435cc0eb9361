#!/bin/bash
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 900 python -u -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 300 python bench.py --steps 3 --warmup 1 --replicas 1 --batch 1 --no-e2e --no-cpu-baseline --candidates 0 --stages > gpurun_out/b_single.json 2> gpurun_out/b_single.err
for RK in "32 4" "32 4" "24 6"; do set -- $RK
  timeout 600 python bench.py --no-cpu-baseline --candidates 0 --no-e2e --steps 6 --replicas $1 --batch $2 > gpurun_out/f_r$1_k$2_$RANDOM.json 2> /dev/null
done
