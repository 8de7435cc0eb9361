"""GPU parity of the tree peel (csrc/fixpoint.cu): the CPD / DFS order of graphs with at
least 2,048 nodes comes from a level-parallel tree construction plus a parallel proof
(general fixed-point rounds when the proof fails, the one-warp peel past the round budget)
instead of the one-warp peel.  Results must equal the reference's peel
(ordering.cpp:40-114) bit for bit through the order API, fuse (the streamed DP then reads a
finished order) and the whole pipeline, single and batched; the context's tree-peel
counters (DP_DEBUG_FIXPOINT) prove which path produced each order.
Cases: layered and shuffled/relabelled graphs (the first tree is proven), rows longer than
64 (global (row, rank) sort), massive cpath ties (rank by id), random DAGs with skip edges
(the proof fails: fixed-point rounds), a zero round budget (the one-warp peel takes over).
"""
import ctypes as C

import numpy as np
import pytest

import paper_2208_00184_b200 as pkg
from cases import GEN, capacity_for, devices
from compare import same, same_graph, same_map, same_pipeline
from graphs import layered, random_dag, shuffled
from paper_2208_00184_b200._abi import Graph

pytestmark = pytest.mark.gpu


@pytest.fixture
def stats(gpu, monkeypatch):
    """Counts of tree-peel outcomes during the test: [proved, rounds, too deep, cycle,
    budget]."""
    monkeypatch.setenv("DP_DEBUG_FIXPOINT", "1")
    lib = pkg.library()

    def read():
        out = (C.c_int64 * 5)()
        lib.dp_ctx_peel_stats(gpu.ctx, out)
        return np.array(out[:], np.int64)
    base = read()
    return lambda: read() - base


def _funnel(seed=3, widths=(12, 6000, 400, 9000, 50, 3000)):
    """Layers of very different widths: nodes of the narrow layers have out-degree in
    the hundreds (rows > 64 take the (row, rank) sort)."""
    rng = np.random.default_rng(seed)
    starts = np.cumsum((0,) + tuple(widths))
    n = int(starts[-1])
    src, dst = [], []
    for li in range(1, len(widths)):
        lo, hi = int(starts[li - 1]), int(starts[li])
        for v in range(int(starts[li]), int(starts[li + 1])):
            k = min(hi - lo, int(rng.integers(2, 7)))
            for u in rng.choice(hi - lo, k, replace=False) + lo:
                src.append(int(u))
                dst.append(v)
    s, d = np.array(src, np.int64), np.array(dst, np.int64)
    o = np.lexsort((d, s))
    return Graph(np.arange(n, dtype=np.int64), rng.integers(100, 901, n), rng.integers(1 << 19, 3 << 19, n), s[o],
                 d[o], rng.integers(1 << 15, 3 << 15, len(s)))


def _orders(gpu, oracle, g, tag):
    _, _, c = oracle.compute_levels(g, GEN)
    same(gpu.cpd_topo(g, c), oracle.cpd_topo(g, c), f"{tag} cpd")
    same(gpu.dfs_topo(g), oracle.dfs_topo(g), f"{tag} dfs")


CASES = {
    "layered": lambda: layered(41, 50000, 5000),
    "layered_deep": lambda: layered(40, 60000, 64),
    "layered_2lv": lambda: layered(42, 20000, 10000),
    "shuffled": lambda: shuffled(layered(43, 30000, 3000), 4, relabel=True),
    "funnel": lambda: _funnel(),
    "ties": lambda: layered(44, 24000, 2000, compute=(7, 7), nbytes=(1000, 1000)),
}


@pytest.fixture(params=["1", "4", "8", "16"])
def cluster(monkeypatch, request):
    """CTAs of the single-graph tree peel's Kahn phase (thread-block cluster; 1 = one CTA)."""
    monkeypatch.setenv("DP_TREE_CLUSTER", request.param)


@pytest.fixture(params=["split", "fused"])
def proof(monkeypatch, request):
    """The proof and emission as grid kernels after the tree kernel (default), or inside it."""
    if request.param == "fused":
        monkeypatch.setenv("DP_TREE_FUSED_PROOF", "1")


@pytest.mark.parametrize("case", sorted(CASES))
def test_tree_orders(gpu, oracle, stats, cluster, proof, case):
    """Every edge joins consecutive levels: the first tree is the peel order."""
    _orders(gpu, oracle, CASES[case](), case)
    assert stats().tolist() == [2, 0, 0, 0, 0]


def test_tree_rounds_random_dag(gpu, oracle, stats, cluster, proof, monkeypatch):
    """Skip edges: the proof fails and fixed-point rounds converge (forced: the cost
    model's budget for these small graphs would hand them to the one-warp peel)."""
    monkeypatch.setenv("DP_PEEL_FIXPOINT", "1")
    _orders(gpu, oracle, random_dag(45, 6000, 0.0006), "random")
    _orders(gpu, oracle, shuffled(random_dag(46, 5000, 0.001), 1, relabel=True), "random_shuffled")
    s = stats()
    assert s[1] >= 3 and s[2:].sum() == 0, s


def test_tree_budget_fallback(gpu, oracle, stats, proof, monkeypatch):
    """No fixed-point rounds allowed: the one-warp peel must produce the order."""
    monkeypatch.setenv("DP_FIXPOINT_ROUNDS", "0")
    monkeypatch.setenv("DP_PEEL_FIXPOINT", "1")
    _orders(gpu, oracle, random_dag(47, 6000, 0.0006), "budget")
    g = random_dag(48, 8000, 0.0005, max_memory=1000)
    total = int(g.memory_bytes.sum())
    ca, ma = gpu.fuse(g, GEN, 200, total // 40)
    cb, mb = oracle.fuse(g, GEN, 200, total // 40)
    same_graph(ca, cb, "fuse")
    same_map(ma, mb, "fuse")
    s = stats()
    assert s[4] >= 3 and s[0] + s[1] == 0, s


def test_tree_gives_up_on_chains(gpu, oracle, stats):
    g = layered(53, 9000, 2, fan_lo=1, fan_hi=2)
    _orders(gpu, oracle, g, "chain")
    assert stats()[2] == 2


@pytest.mark.parametrize("r", [1, 33, 200, 256])
def test_tree_fuse(gpu, oracle, r):
    """fuse on a tree-peeled graph: the streamed DP runs on a finished order."""
    g = layered(49, 60000, 6000)
    total = int(g.memory_bytes.sum())
    for limit in (total // 8, total // 500):
        ca, ma = gpu.fuse(g, GEN, r, limit)
        cb, mb = oracle.fuse(g, GEN, r, limit)
        same_graph(ca, cb, f"r{r}")
        same_map(ma, mb, f"r{r}")


def test_tree_pipeline_single_and_batch(gpu, ref):
    gs = [layered(50, 40000, 8000), _funnel(51), shuffled(layered(52, 20000, 4000), 5, relabel=True),
          layered(54, 30000, 300)]
    devs = devices(8, max(capacity_for(g, 8, 1.25) for g in gs))
    want = [ref.evaluate_pipeline(g, devs, GEN) for g in gs]
    for i, (g, w) in enumerate(zip(gs, want)):
        same_pipeline(gpu.evaluate_pipeline(g, devs, GEN), w, f"single[{i}]")
    for i, r in enumerate(gpu.evaluate_pipeline_batch(gs, devs, GEN)):
        same_pipeline(r, want[i], f"batch[{i}]")
