"""Small workloads that launch every hot kernel once, for compute-sanitizer
(memcheck / racecheck / synccheck) on the GPU box:

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py

k_peel_dp (pair), k_peel_dp_shared (batch of graphs), k_levels_flow, k_levels_seq, k_peel2,
k_place, k_sim / k_sim_wide; each result is checked against the oracle restatement."""
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
print("sanitize probe ok", flush=True)
