"""Seeded graph families for the parity suites (numpy; test inputs only).

random_dag follows the shape of the reference's property-test fixture
(tests/support/test_util.hpp:131-151: spanning parent + Bernoulli extra edges);
layered follows SURVEY §8(d)'s layered recipe shape (fan-in from the previous layer).
Exact RNG streams differ from std::mt19937_64 — these are inputs fed identically to
every implementation, not reproductions of the reference's own fixtures.
"""
from __future__ import annotations

import numpy as np

from paper_2208_00184_b200._abi import Graph


def random_dag(seed: int, n: int, extra_p: float, max_compute=50, max_memory=100, max_bytes=80,
               min_compute=1, min_memory=1, min_bytes=0) -> Graph:
    rng = np.random.default_rng(seed)
    ids = np.arange(n, dtype=np.int64)
    comp = rng.integers(min_compute, max_compute + 1, n)
    mem = rng.integers(min_memory, max_memory + 1, n)
    src, dst = [], []
    for v in range(1, n):
        u = int(rng.integers(0, v))
        src.append(u)
        dst.append(v)
        if extra_p > 0:
            extra = np.nonzero(rng.random(v) < extra_p)[0]
            for w in extra:
                if w != u:
                    src.append(int(w))
                    dst.append(v)
    m = len(src)
    b = rng.integers(min_bytes, max_bytes + 1, m)
    return Graph(ids, comp, mem, np.array(src, np.int64), np.array(dst, np.int64), b)


def layered(seed: int, n: int, width: int, fan_lo=2, fan_hi=6, compute=(100, 900),
            memory=(1 << 19, 3 << 19), nbytes=(1 << 15, 3 << 15), sort_edges=True) -> Graph:
    rng = np.random.default_rng(seed)
    ids = np.arange(n, dtype=np.int64)
    comp = rng.integers(compute[0], compute[1] + 1, n)
    mem = rng.integers(memory[0], memory[1] + 1, n)
    src, dst = [], []
    for v in range(width, n):
        layer = v // width
        lo = (layer - 1) * width
        hi = min(lo + width, n)
        k = min(hi - lo, int(rng.integers(fan_lo, fan_hi + 1)))
        picks = rng.choice(hi - lo, size=k, replace=False) + lo
        src.extend(picks.tolist())
        dst.extend([v] * k)
    s = np.array(src, np.int64)
    d = np.array(dst, np.int64)
    if sort_edges:
        o = np.lexsort((d, s))
        s, d = s[o], d[o]
    b = rng.integers(nbytes[0], nbytes[1] + 1, len(s))
    return Graph(ids, comp, mem, s, d, b)


def shuffled(g: Graph, seed: int, relabel: bool = False) -> Graph:
    """Permute node and edge order (test_util.hpp:153-159); optionally remap ids to
    sparse, non-dense int64 values so the id->index sort path is exercised."""
    rng = np.random.default_rng(seed)
    pn = rng.permutation(g.n)
    pe = rng.permutation(g.m)
    ids, src, dst = g.node_id, g.edge_src, g.edge_dst
    if relabel:
        newid = rng.choice(np.int64(1) << 40, size=g.n, replace=False).astype(np.int64) - (np.int64(1) << 39)
        lut = dict(zip(g.node_id.tolist(), newid.tolist()))
        ids = newid
        src = np.array([lut[x] for x in g.edge_src.tolist()], np.int64)
        dst = np.array([lut[x] for x in g.edge_dst.tolist()], np.int64)
    grp = None if g.group is None else g.group[pn]
    return Graph(ids[pn], g.compute_us[pn], g.memory_bytes[pn], src[pe], dst[pe], g.edge_bytes[pe], grp)


def with_groups(g: Graph, seed: int, n_groups: int, frac: float) -> Graph:
    rng = np.random.default_rng(seed)
    grp = np.full(g.n, -1, np.int32)
    pick = rng.random(g.n) < frac
    grp[pick] = rng.integers(0, n_groups, int(pick.sum()))
    return Graph(g.node_id, g.compute_us, g.memory_bytes, g.edge_src, g.edge_dst, g.edge_bytes, grp)


def chain(costs, nbytes) -> Graph:
    n = len(costs)
    return Graph.make([(i, costs[i]) for i in range(n)], [(i, i + 1, nbytes[i]) for i in range(n - 1)])
