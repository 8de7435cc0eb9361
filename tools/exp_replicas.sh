mkdir -p gpurun_out
for R in 1 2 4 8 16 32 64; do
  timeout 300 python bench.py --steps 2 --warmup 1 --replicas $R --no-e2e --no-cpu-baseline --candidates 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print($R, d['ms_per_step'], d['value']/1e6, d['single_graph']['ms'])" >> gpurun_out/exp_replicas.txt
done
