"""Parity case catalogue: the reference tests' hand goldens (cited), seeded property
families, and the invalid inputs the reference's validate() distinguishes."""
from __future__ import annotations

import numpy as np

from paper_2208_00184_b200._abi import Graph
from graphs import chain, layered, random_dag, shuffled, with_groups

UNIT = (1.0, 0.0)          # test_util.hpp:46
GEN = (0.001, 10.0)        # generator.hpp:33
HALF = (0.5, 0.5)          # exercises llround half-away-from-zero
ODD = (0.1, 0.25)


def golden_graphs():
    """Hand-computed fixtures from /root/reference/proj/tests."""
    return {
        # test_graph_core.cpp:93-103 chain: t{0,7,12} b{13,6,1}
        "chain3": chain([2, 3, 1], [5, 2]),
        # test_ordering.cpp:58-62 / test_graph_core.cpp:112-117 diamond
        "diamond": Graph.make([(0, 1), (1, 1), (2, 1), (3, 1)],
                              [(0, 1, 1), (0, 2, 1), (1, 3, 1), (2, 3, 1)]),
        # test_ordering.cpp:15-27 two_chains(4)
        "two_chains": Graph.make([(c * 4 + i, 1) for c in range(2) for i in range(4)],
                                 [(c * 4 + i - 1, c * 4 + i, 10) for c in range(2) for i in range(1, 4)]),
        # test_ordering.cpp:36-39 sources FIFO
        "sources_fifo": Graph.make([(1, 1), (2, 1), (3, 1)], [(1, 3, 1), (2, 3, 1)]),
        "single": Graph.make([(7, 5)], []),
        "empty": Graph.make([], []),
        "isolated": Graph.make([(5, 1), (3, 2), (9, 0)], []),
        # fusion chain4 (test_fusion.cpp:59-71 shape)
        "chain4": chain([1, 1, 1, 1], [10, 1, 10]),
        # simulator send-engine tie (test_simulator.cpp:118-133 shape)
        "fanout": Graph.make([(0, 2), (1, 1), (2, 1)], [(0, 1, 5), (0, 2, 5)]),
    }


def valid_families(scale: int = 1):
    out = dict(golden_graphs())
    for s in range(6):
        out[f"rdag{s}"] = random_dag(100 + s, 5 + 7 * s, 0.15 if s % 2 else 0.05)
    out["rdag_zero"] = random_dag(7, 40, 0.1, min_compute=0, max_compute=3, min_bytes=0, max_bytes=2)
    out["layered_small"] = layered(3, 400 * scale, 16)
    out["layered_wide"] = layered(4, 600 * scale, 150, fan_lo=1, fan_hi=3)
    out["layered_deep"] = layered(5, 500 * scale, 4, fan_lo=1, fan_hi=4)
    out["shuf"] = shuffled(random_dag(11, 50, 0.1), 3)
    out["shuf_relabel"] = shuffled(layered(12, 300, 10), 4, relabel=True)
    out["groups"] = with_groups(random_dag(21, 40, 0.05), 5, 6, 0.4)
    out["groups_layered"] = with_groups(layered(22, 300, 12), 6, 30, 0.2)
    return out


def invalid_graphs():
    g = lambda nodes, edges: Graph.make(nodes, edges)  # noqa: E731
    return {
        "dup_id": g([(0, 1), (1, 1), (0, 2)], [(0, 1, 1)]),
        "dangling": g([(0, 1), (1, 1)], [(0, 5, 1), (7, 1, 2)]),
        "self_loop": g([(0, 1), (1, 1)], [(0, 1, 1), (1, 1, 1)]),
        "neg_compute": g([(0, -1), (1, 1)], [(0, 1, 1)]),
        "neg_memory": g([(0, 1, -5), (1, 1)], [(0, 1, 1)]),
        "neg_bytes": g([(0, 1), (1, 1)], [(0, 1, -1)]),
        "parallel": g([(0, 1), (1, 1), (2, 1)], [(0, 1, 1), (1, 2, 1), (0, 1, 3), (0, 1, 4)]),
        "cycle2": g([(0, 1), (1, 1)], [(0, 1, 1), (1, 0, 1)]),
        "cycle_tail": g([(0, 1), (1, 1), (2, 1), (3, 1), (4, 1)],
                        [(0, 1, 1), (1, 2, 1), (2, 3, 1), (3, 1, 1), (3, 4, 1)]),
        "many": g([(0, -1, -1), (0, 1), (1, 1), (2, 1)],
                  [(0, 1, -2), (1, 9, 1), (2, 2, 1), (0, 1, 1), (1, 2, 1), (2, 1, 1)]),
    }


def devices(d: int, cap: int, shuffle_seed: int | None = None, base_id: int = 0, stride: int = 1):
    ids = [base_id + stride * i for i in range(d)]
    devs = [(i, cap) for i in ids]
    if shuffle_seed is not None:
        rng = np.random.default_rng(shuffle_seed)
        devs = [devs[i] for i in rng.permutation(d)]
    return devs


def capacity_for(g: Graph, d: int, factor: float = 1.25) -> int:
    total = int(g.memory_bytes.sum()) if g.n else 1
    return max(1, int(factor * total / d))
