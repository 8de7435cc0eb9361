"""Pin the plain-C oracle (oracle/dp_oracle.c) to the UNMODIFIED reference
(oracle/_ref/libdagplace_ref.so, built from /root/reference/proj/src by oracle/Makefile).

Every function of the hot path is run on both over the reference tests' hand goldens,
seeded property families and the invalid inputs validate() distinguishes; results and
errors (kind + message text) must be identical.  Also checks the literal golden values
of the reference's own tests so the oracle is pinned even where _ref is absent."""
import numpy as np
import pytest

import parity
from cases import GEN, UNIT, golden_graphs, invalid_graphs, valid_families
from graphs import layered, random_dag

VALID = valid_families()
INVALID = invalid_graphs()


@pytest.mark.parametrize("name", sorted(VALID) + sorted(INVALID))
def test_core_pinned(oracle, ref, name):
    g = VALID.get(name) or INVALID[name]
    parity.check_core(oracle, ref, g, name)


@pytest.mark.parametrize("name", sorted(VALID))
def test_fusion_pinned(oracle, ref, name):
    parity.check_fusion(oracle, ref, VALID[name], name)


@pytest.mark.parametrize("name", sorted(VALID))
def test_placement_pinned(oracle, ref, name):
    parity.check_placement(oracle, ref, VALID[name], name)


@pytest.mark.parametrize("name", sorted(VALID))
def test_simulate_pinned(oracle, ref, name):
    parity.check_simulate(oracle, ref, VALID[name], name)


@pytest.mark.parametrize("name", sorted(VALID))
def test_pipeline_pinned(oracle, ref, name):
    parity.check_pipeline(oracle, ref, VALID[name], name)


def test_candidates_and_bruteforce_pinned(oracle, ref):
    g = random_dag(5, 9, 0.2, max_bytes=30)
    devs = [(4, 10 ** 6), (1, 10 ** 6), (9, 10 ** 6)]
    a = oracle.brute_force_optimal(g, devs, UNIT)
    b = ref.brute_force_optimal(g, devs, UNIT)
    assert a[1] == b[1]
    assert np.array_equal(a[0], b[0])
    rng = np.random.default_rng(0)
    ncl = 4
    node_cluster = rng.integers(0, ncl, g.n).astype(np.int32)
    cand = rng.integers(0, 3, (50, ncl)).astype(np.uint8)
    ma, ia = oracle.simulate_candidates(g, node_cluster, ncl, cand, devs, GEN)
    mb, ib = ref.simulate_candidates(g, node_cluster, ncl, cand, devs, GEN, threads=2)
    assert np.array_equal(ma, mb) and ia == ib


def test_literal_goldens(oracle):
    """Literal values asserted by the reference's own tests (file:line cited)."""
    G = golden_graphs()
    # test_graph_core.cpp:66-77 comm_time
    assert oracle.comm_time(7, UNIT) == 7
    assert oracle.comm_time(10, (2.0, 7.0)) == 27
    assert oracle.comm_time(2, (0.5, 0.0)) == 1 and oracle.comm_time(3, (0.5, 0.0)) == 2
    assert oracle.comm_time(1, (0.5, 0.0)) == 1  # llround(0.5) = 1 (half away from zero)
    # test_graph_core.cpp:93-103 chain levels
    t, b, c = oracle.compute_levels(G["chain3"], UNIT)
    assert t.tolist() == [0, 7, 12] and b.tolist() == [13, 6, 1] and c.max() == 13
    # test_graph_core.cpp:112-117 diamond cpath 5
    assert oracle.compute_levels(G["diamond"], UNIT)[2].max() == 5
    # test_ordering.cpp:44-56
    assert oracle.m_topo(G["two_chains"]).tolist() == [0, 4, 1, 5, 2, 6, 3, 7]
    assert oracle.dfs_topo(G["two_chains"]).tolist() == list(range(8))
    assert oracle.m_topo(G["sources_fifo"]).tolist() == [1, 2, 3]
    # test_fusion.cpp:59-71 chain4 clusters {0,1},{2,3}, breakpoints {2}
    g4 = G["chain4"]
    seq = oracle.dfs_topo(g4)
    m = oracle.optimal_breakpoints(g4, seq, UNIT, 2, 100)
    assert [x.tolist() for x in m.members] == [[0, 1], [2, 3]] and m.breakpoints.tolist() == [2]
    # test_simulator.cpp:118-133: sends end at 7 and 12, makespan 13
    r = oracle.simulate(G["fanout"], np.array([0, 1, 1], np.int32), [(0, 100), (1, 100)], UNIT, True)
    tr = r.trace
    sends = {int(d): int(e) for k, d, e in zip(tr["kind"], tr["dst"], tr["end"]) if k == 1}
    assert sends == {1: 7, 2: 12} and r.makespan == 13
    # test_simulator.cpp:95-104 split chain 10; :106-116 diamond 5
    g2 = G["chain3"]
    assert oracle.simulate(g2, np.array([0, 0, 0], np.int32), [(0, 100)], UNIT).makespan == 6
    rd = oracle.simulate(G["diamond"], np.array([0, 0, 1, 0], np.int32), [(0, 100), (1, 100)], UNIT)
    assert rd.makespan == 5 and rd.cross_transfer_count == 2
    # test_placement.cpp:55-67 order_place golden
    g = __import__("paper_2208_00184_b200._abi", fromlist=["Graph"]).Graph.make(
        [(0, 1, 40), (1, 1, 40), (2, 1, 40), (3, 1, 40)], [(0, 1, 1), (1, 2, 1), (2, 3, 1)])
    p = oracle.order_place(g, oracle.dfs_topo(g), [(0, 100), (1, 100)])
    assert p.device.tolist() == [0, 0, 1, 1] and p.per_device_memory.tolist() == [80, 80]
    assert not p.oom_risk


@pytest.mark.slow
def test_pipeline_pinned_medium(oracle, ref):
    g = layered(77, 20000, 64)
    parity.check_pipeline(oracle, ref, g, "layered20k", d=8)
