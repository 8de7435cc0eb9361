"""Small workloads that launch every hot kernel once, for compute-sanitizer
(memcheck / racecheck / synccheck) on the GPU box:

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py

k_peel_dp (pair), k_peel_dp_shared (batch of graphs), k_levels_flow_batch (narrow and wide
plans), k_levels_seq, k_peel2 (v5 and v6 dense), k_treepeel (one CTA and the 16-CTA cluster),
k_rs_hist / k_rs_scatter / scans (dense and sorted ids), k_traceback, k_place, k_sim /
k_sim_wide; each result is checked against the oracle restatement."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_2208_00184_b200 as pkg  # noqa: E402
from cases import GEN, capacity_for, devices  # noqa: E402
from compare import same, same_pipeline, same_sim  # noqa: E402
from graphs import layered  # noqa: E402
from oracle.bind import oracle_backend  # noqa: E402

gpu, ora = pkg.device(0), oracle_backend()
g = layered(5, 20000, 64)
devs = devices(8, capacity_for(g, 8, 1.25))
same_pipeline(gpu.evaluate_pipeline(g, devs, GEN), ora.evaluate_pipeline(g, devs, GEN), "pair")
gs = [layered(6 + i, 8000, 32) for i in range(3)]
for a, b in zip(gpu.evaluate_pipeline_batch(gs, devs, GEN), [ora.evaluate_pipeline(x, devs, GEN) for x in gs]):
    same_pipeline(a, b, "shared")
for x, y in zip(gpu.compute_levels(g, GEN), ora.compute_levels(g, GEN)):
    same(x, y, "levels")
_, _, cp = ora.compute_levels(g, GEN)
same(gpu.cpd_topo(g, cp), ora.cpd_topo(g, cp), "cpd")
ids = np.array(sorted(d for d, _ in devs), np.int32)
place = ids[np.random.default_rng(1).integers(0, 8, g.n)]
same_sim(gpu.simulate(g, place, devs, GEN, True), ora.simulate(g, place, devs, GEN, True), "sim")
d16 = devices(16, capacity_for(g, 16, 1.25))
ids16 = np.array(sorted(d for d, _ in d16), np.int32)
p16 = ids16[np.random.default_rng(2).integers(0, 16, g.n)]
same_sim(gpu.simulate(g, p16, d16, GEN, False), ora.simulate(g, p16, d16, GEN, False), "sim16")
# round 2: wide dataflow plan + cluster tree peel (mean edge span >= 8,192), relabelled ids
# (radix sort of the id index), the one-warp peel in dense mode
from graphs import shuffled  # noqa: E402
gw = layered(9, 40000, 20000)
for x, y in zip(gpu.compute_levels(gw, GEN), ora.compute_levels(gw, GEN)):
    same(x, y, "levels wide")
_, _, cw = ora.compute_levels(gw, GEN)
same(gpu.cpd_topo(gw, cw), ora.cpd_topo(gw, cw), "cpd wide (cluster)")
gr = shuffled(layered(10, 12000, 200), 3, relabel=True)
for x, y in zip(gpu.compute_levels(gr, GEN), ora.compute_levels(gr, GEN)):
    same(x, y, "levels relabelled")
os.environ["DP_PEEL_NO_FIXPOINT"] = "1"
gd = layered(11, 6000, 60, fan_lo=30, fan_hi=50)
_, _, cd = ora.compute_levels(gd, GEN)
same(gpu.cpd_topo(gd, cd), ora.cpd_topo(gd, cd), "cpd v6 dense")
del os.environ["DP_PEEL_NO_FIXPOINT"]
print("sanitize probe ok", flush=True)
