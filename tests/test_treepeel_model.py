"""CPU pinning of the tree-peel algorithm (csrc/fixpoint.cu) through its Python model
(tests/treepeel_model.py): on seeded families the model's order equals the oracle's
cpd_topo / dfs_topo (ordering.cpp:40-114) exactly, and on layered DAGs (every edge joins
consecutive levels, the config #4 shape) the first tree already passes the proof."""
import numpy as np
import pytest

from graphs import layered, random_dag, shuffled
from treepeel_model import ranks_cpd, ranks_dfs, tree_peel

GEN = (0.001, 10.0)


def _index(g):
    idx = {int(x): i for i, x in enumerate(g.node_id.tolist())}
    src = [idx[int(x)] for x in g.edge_src.tolist()]
    dst = [idx[int(x)] for x in g.edge_dst.tolist()]
    return src, dst


def _check(oracle, g, expect_first=None):
    src, dst = _index(g)
    _, _, c = oracle.compute_levels(g, GEN)
    for name, rank, want in (("cpd", ranks_cpd(c, g.node_id), oracle.cpd_topo(g, c)),
                             ("dfs", ranks_dfs(g.node_id), oracle.dfs_topo(g))):
        order, first, rounds = tree_peel(g.n, src, dst, rank)
        got = g.node_id[np.array(order, np.int64)]
        assert np.array_equal(got, want), name
        if expect_first is not None:
            assert first == expect_first, (name, rounds)


@pytest.mark.parametrize("seed,n,w", [(1, 400, 20), (2, 900, 300), (3, 600, 7), (4, 300, 150)])
def test_model_layered_one_tree(oracle, seed, n, w):
    _check(oracle, layered(seed, n, w), expect_first=True)
    _check(oracle, shuffled(layered(seed + 10, n, w), seed, relabel=True), expect_first=True)


@pytest.mark.parametrize("seed,p", [(5, 0.0), (6, 0.01), (7, 0.05), (8, 0.2)])
def test_model_random_dags(oracle, seed, p):
    """Skip edges across levels: the proof may fail and the general rounds converge."""
    _check(oracle, random_dag(seed, 300, p))
    _check(oracle, shuffled(random_dag(seed + 20, 250, p), seed), None)


def test_model_ties(oracle):
    g = layered(9, 500, 25, compute=(5, 5), nbytes=(100, 100))
    _check(oracle, g, expect_first=True)
