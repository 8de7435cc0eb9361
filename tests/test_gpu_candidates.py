"""Config #5 (BASELINE.json): a batch of candidate placements of the 100k-op DAG, makespans
on the GPU (dp_simulate_candidates, one warp per candidate) against the UNMODIFIED
reference — a loop of simulate() (simulator.cpp:56-252) with the first-strict-minimum
argmin of brute_force_optimal (simulator.cpp:292-294).

* candidates 0..511 bit-exact against tests/golden/candidates5.json (made by
  tests/golden/make_golden.py --candidates from oracle/_ref);
* the full 65,536-candidate batch: the argmin and a spread sample re-checked against the
  oracle restatement;
* the engine-ring overflow -> re-run path forced (DP_SIM_QUEUE) with identical results."""
import json
import os

import numpy as np
import pytest

from golden.make_golden import digest
from golden_configs import config5_candidates

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "candidates5.json")))


@pytest.fixture(scope="module")
def c5(gpu):
    return config5_candidates(gpu, 0, GOLD["count"])


def test_config5_prefix_matches_reference(gpu, c5):
    g, devs, comm, rep, cand = c5
    assert digest(cand) == GOLD["rows_digest"], "candidate family drifted"
    ms, am = gpu.simulate_candidates(g, rep.map.node_cluster, rep.coarse_nodes, cand, devs, comm)
    assert [int(x) for x in ms] == GOLD["makespans"]
    assert am == GOLD["argmin"]


def test_config5_full_batch(gpu, oracle, c5):
    from paper_2208_00184_b200 import synth
    g, devs, comm, rep, cand0 = c5
    B = 65536
    base = cand0[0]
    cand = synth.candidates(base, len(devs), 0, B)
    assert np.array_equal(cand[:GOLD["count"]], cand0)
    ms, am = gpu.simulate_candidates(g, rep.map.node_cluster, rep.coarse_nodes, cand, devs, comm)
    assert [int(x) for x in ms[:GOLD["count"]]] == GOLD["makespans"]
    assert am == int(np.argmin(ms)) and ms[am] == ms.min()  # np.argmin: first minimum
    # the winner and a spread sample against the oracle restatement
    pick = sorted({am, B - 1, *range(GOLD["count"], B, 4099)})
    mo, _ = oracle.simulate_candidates(g, rep.map.node_cluster, rep.coarse_nodes, cand[pick], devs, comm)
    assert [int(x) for x in ms[pick]] == [int(x) for x in mo]


@pytest.mark.parametrize("q", ["1", "4", "16"])
def test_ring_overflow_rerun(gpu, oracle, monkeypatch, q):
    """First-pass rings of q entries overflow on most candidates; the re-run (16x larger
    rings, up to the exact bound) must give the same makespans."""
    from cases import GEN
    from graphs import layered
    g = layered(31, 3000, 48)
    _, m = oracle.fuse(g, GEN, 200, int(g.memory_bytes.sum()) // 16)
    rng = np.random.default_rng(int(q))
    cand = rng.integers(0, 8, (40, m.n_clusters)).astype(np.uint8)
    devs = [(d, 10 ** 12) for d in range(8)]
    want, wam = oracle.simulate_candidates(g, m.node_cluster, m.n_clusters, cand, devs, GEN)
    monkeypatch.setenv("DP_SIM_QUEUE", q)
    got, gam = gpu.simulate_candidates(g, m.node_cluster, m.n_clusters, cand, devs, GEN)
    assert [int(x) for x in got] == [int(x) for x in want] and gam == wam
    ids = np.arange(8, dtype=np.int32)
    place = ids[cand[3][m.node_cluster]]
    a = gpu.simulate(g, place, devs, GEN, True)
    b = oracle.simulate(g, place, devs, GEN, True)
    from compare import same_sim
    same_sim(a, b, f"overflow q{q}")
