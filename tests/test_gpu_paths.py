"""GPU parity for the special paths of the sequential kernels (peel_dp.cu, graph.cu):
each case is built to force one code path and is compared bit-exactly with the oracle
restatement (oracle/dp_oracle.c).

  peel v6        in-degree >= 127 (global counters), out-degree > 8 (CSR rows), full
                 hash buckets (global spill counters), DFS as well as CPD ranks
                 (the tree peel of fixpoint.cu is switched off where the one-warp peel's
                 path is the point; test_gpu_fixpoint.py covers the tree peel)
  streamed DP    v3 (R <= 225), 32-step blocks (226..256), per-step 32-bit keys (cost
                 bound), 64-bit keys (large costs), R = 1 / 32 / 33 block edges
  levels         index-order sweep (n <= 16384, index order topological) vs the Kahn
                 frontier (shuffled ids, n just above the sweep limit)
"""
import numpy as np
import pytest

from compare import same, same_graph, same_map
from graphs import layered, shuffled
from paper_2208_00184_b200._abi import Graph

pytestmark = pytest.mark.gpu

GEN = (0.001, 10.0)


def _fanin_hub(seed=5, hubs=3, preds=200, n=2000):
    """Nodes with in-degree `preds` (>= 127) among an otherwise layered DAG."""
    rng = np.random.default_rng(seed)
    g = layered(seed, n, 40)
    src, dst = list(g.edge_src), list(g.edge_dst)
    for h in range(hubs):
        v = n - 1 - h
        layer_lo = (v // 40 - 1) * 40
        cand = np.setdiff1d(np.arange(0, layer_lo), np.array(src)[np.array(dst) == v])
        for u in rng.choice(cand, preds, replace=False):
            src.append(int(u))
            dst.append(v)
    o = np.lexsort((dst, src))
    s, d = np.array(src)[o], np.array(dst)[o]
    return Graph(g.node_id, g.compute_us, g.memory_bytes, s, d, rng.integers(1 << 15, 3 << 15, len(s)))


def _orders(gpu, oracle, g):
    t, b, c = oracle.compute_levels(g, GEN)
    same(gpu.cpd_topo(g, c), oracle.cpd_topo(g, c), "cpd")
    same(gpu.dfs_topo(g), oracle.dfs_topo(g), "dfs")
    a = gpu.compute_levels(g, GEN)
    for x, y, nm in zip(a, (t, b, c), "tbc"):
        same(x, y, nm)


@pytest.fixture(params=["dense", "hash"])
def warp_peel(monkeypatch, request):
    """The one-warp peel's special paths are the point: no tree peel first; remaining
    in-degrees as dense 16-bit counters (graphs up to 81,920 nodes) or in the hash table."""
    monkeypatch.setenv("DP_PEEL_NO_FIXPOINT", "1")
    if request.param == "hash":
        monkeypatch.setenv("DP_PEEL_NO_DENSE", "1")


def test_peel_high_indegree(gpu, oracle, warp_peel):
    _orders(gpu, oracle, _fanin_hub())


@pytest.mark.parametrize("v6", [None, "1"])
def test_peel_long_rows(gpu, oracle, warp_peel, monkeypatch, v6):
    # fan-out up to 30 from the previous layer: many rows longer than 8 (v5's 32-slot rows,
    # or v6's CSR path with dense counters when forced)
    if v6:
        monkeypatch.setenv("DP_PEEL_V6_DENSE", v6)
    g = layered(9, 6000, 60, fan_lo=6, fan_hi=30)
    _orders(gpu, oracle, g)


def test_peel_v6_dense_wide_rows(gpu, oracle, warp_peel):
    # more than 32 children per node on average: v6 in dense mode by default (hash mode: v5)
    _orders(gpu, oracle, layered(19, 8000, 200, fan_lo=30, fan_hi=60))


@pytest.mark.parametrize("n", [81920, 81921])
def test_peel_dense_limit(gpu, oracle, warp_peel, n):
    # the dense mode's node limit (k_peel2: 2 x (2^15 + 2^13) counters) and one past it
    _orders(gpu, oracle, layered(17, n, 3000, fan_lo=2, fan_hi=12))


def test_peel_dense_huge_indegree(gpu, oracle, warp_peel):
    # an in-degree of 65,535 does not fit a 16-bit counter: the peel falls back to the table
    n = 66000
    rng = np.random.default_rng(4)
    src = np.concatenate([np.arange(65535), np.arange(65535, n - 1)])
    dst = np.concatenate([np.full(65535, n - 1), np.arange(65536, n)])
    o = np.lexsort((dst, src))
    g = Graph(np.arange(n), rng.integers(1, 100, n), np.ones(n, np.int64), src[o], dst[o],
              rng.integers(0, 1 << 20, n - 1))
    _orders(gpu, oracle, g)


def test_peel_bucket_spill(gpu, oracle, warp_peel):
    # a 40k-wide layer keeps tens of thousands of nodes open: buckets overflow to HBM
    g = layered(13, 120000, 40000, fan_lo=2, fan_hi=5)
    _orders(gpu, oracle, g)


@pytest.mark.parametrize("r", [1, 2, 31, 32, 33, 200, 224, 225, 226, 256])
def test_streamed_dp_ranges(gpu, oracle, r):
    g = layered(17, 12000, 48)
    total = int(g.memory_bytes.sum())
    for limit in (total // 4, total // 300):
        ca, ma = gpu.fuse(g, GEN, r, limit)
        cb, mb = oracle.fuse(g, GEN, r, limit)
        same_graph(ca, cb, f"r{r}")
        same_map(ma, mb, f"r{r}")


@pytest.mark.parametrize("scale", [1 << 20, 1 << 26, 1 << 40])
def test_streamed_dp_cost_widths(gpu, oracle, scale):
    """Costs sized to select the per-step 32-bit path (block bound fails) and the 64-bit
    path (32-bit keys cannot hold the window)."""
    g = layered(23, 6000, 32, nbytes=(scale, 2 * scale))
    total = int(g.memory_bytes.sum())
    for r in (20, 200):
        ca, ma = gpu.fuse(g, GEN, r, total // 6)
        cb, mb = oracle.fuse(g, GEN, r, total // 6)
        same_graph(ca, cb, f"s{scale} r{r}")
        same_map(ma, mb, f"s{scale} r{r}")


@pytest.mark.parametrize("n", [16383, 16384, 16385])
def test_levels_indexorder_limit(gpu, oracle, n):
    g = layered(29, n, 3, fan_lo=1, fan_hi=3)
    a = gpu.compute_levels(g, GEN)
    b = oracle.compute_levels(g, GEN)
    for x, y, nm in zip(a, b, "tbc"):
        same(x, y, nm)
    h = shuffled(g, 3, relabel=True)  # index order no longer topological: Kahn path
    a = gpu.compute_levels(h, GEN)
    b = oracle.compute_levels(h, GEN)
    for x, y, nm in zip(a, b, "tbc"):
        same(x, y, nm)


def test_levels_indexorder_long_row(gpu, oracle):
    # one node with more in-edges than a staged tile (8,192 edges): the sweep reads it from HBM
    n = 12000
    rng = np.random.default_rng(2)
    src = list(range(9000)) + list(rng.integers(0, 11000, 3000))
    dst = [11999] * 9000 + [int(x) + 1 + int(rng.integers(0, 999)) for x in rng.integers(0, 11000, 3000)]
    pairs = sorted({(s, d) for s, d in zip(src, dst) if s < d < n})
    g = Graph(np.arange(n), rng.integers(1, 100, n), np.ones(n, np.int64), [p[0] for p in pairs],
              [p[1] for p in pairs], rng.integers(0, 1 << 20, len(pairs)))
    a = gpu.compute_levels(g, GEN)
    b = oracle.compute_levels(g, GEN)
    for x, y, nm in zip(a, b, "tbc"):
        same(x, y, nm)


def _levels_same(gpu, oracle, g):
    a = gpu.compute_levels(g, GEN)
    b = oracle.compute_levels(g, GEN)
    for x, y, nm in zip(a, b, "tbc"):
        same(x, y, nm)


@pytest.mark.parametrize("warps", [None, "1", "64"])
@pytest.mark.parametrize("shape", ["deep", "wide", "chain", "hub", "long_rows"])
def test_levels_dataflow(gpu, oracle, monkeypatch, shape, warps):
    """Index-topological graphs above the sweep limit take the dataflow kernel
    (k_levels_flow_batch): deep and wide layers, a near-chain (inputs inside the warp's own
    chunk), in-degree hubs, rows > 8; with the default warp count, one warp per SM per pass
    and more warps than fit on the GPU at once (tickets are only taken by running warps)."""
    if warps is not None:
        monkeypatch.setenv("DP_FLOW_WARPS", warps)
    g = {"deep": lambda: layered(31, 60000, 500),
         "wide": lambda: layered(32, 80000, 20000),
         "chain": lambda: layered(33, 20000, 2, fan_lo=1, fan_hi=2),
         "hub": lambda: _fanin_hub(7, hubs=4, preds=300, n=20000),
         "long_rows": lambda: layered(34, 30000, 100, fan_lo=8, fan_hi=30)}[shape]()
    _levels_same(gpu, oracle, g)


@pytest.mark.parametrize("grain", ["1", "3", "8"])
@pytest.mark.parametrize("ahead", ["1", "3", "100000"])
def test_levels_dataflow_lookahead(gpu, oracle, monkeypatch, ahead, grain):
    # the lookahead only throttles ticket holders and a ticket's grain only groups chunks:
    # any values must give the same levels
    monkeypatch.setenv("DP_FLOW_AHEAD", ahead)
    monkeypatch.setenv("DP_FLOW_GRAIN", grain)
    _levels_same(gpu, oracle, layered(35, 40000, 700))


@pytest.mark.parametrize("case", ["r32", "r225", "r226", "wide_cost", "spill", "hub"])
def test_shared_sm_mode(gpu, oracle, monkeypatch, case):
    """The one-SM-per-graph peel + DP kernel used by batched calls (k_peel_dp_shared:
    8,192 hash buckets, 1,024 staged in-edges per chunk), forced for single graphs."""
    monkeypatch.setenv("DP_PEEL_DP_SHARED", "1")
    monkeypatch.setenv("DP_PEEL_NO_FIXPOINT", "1")
    if case == "spill":
        g, r = layered(13, 120000, 40000, fan_lo=2, fan_hi=5), 200
    elif case == "hub":
        g, r = _fanin_hub(11, hubs=3, preds=400, n=20000), 150
    elif case == "wide_cost":
        g, r = layered(23, 6000, 32, nbytes=(1 << 26, 2 << 26)), 200
    else:
        g, r = layered(17, 12000, 48, fan_lo=4, fan_hi=12), int(case[1:])
    total = int(g.memory_bytes.sum())
    for limit in (total // 4, total // 300):
        ca, ma = gpu.fuse(g, GEN, r, limit)
        cb, mb = oracle.fuse(g, GEN, r, limit)
        same_graph(ca, cb, case)
        same_map(ma, mb, case)
