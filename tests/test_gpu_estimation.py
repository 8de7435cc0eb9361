"""GPU parity of the Standard Evaluation kernels (estimation.cu) with the UNMODIFIED
reference's estimation.cpp (oracle/_ref): fp64 fits, estimated graphs, the fitted comm
model and the deviation report are compared BIT-exactly (numpy array_equal on float64),
errors by kind and message."""
import numpy as np
import pytest

from paper_2208_00184_b200._abi import DagError, Estimation, Graph, Profiles
from graphs import layered, random_dag

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def est(gpu, ref):
    return Estimation(gpu.lib, "dp_", ctx=gpu.ctx), Estimation(ref.lib, "dpr_")


def _profiles(rng, ids, batches, noise=True, shuffle=True):
    bs, off, nid, mem, tim = [], [0], [], [], []
    for b in batches:
        order = rng.permutation(len(ids)) if shuffle else np.arange(len(ids))
        for i in order:
            base_m = 1000 + 37 * (ids[i] % 97)
            base_t = 10 + (ids[i] % 13)
            nid.append(ids[i])
            mem.append(int(base_m * b + (rng.integers(-50, 50) if noise else 0)))
            tim.append(int(base_t * b // 3 + (rng.integers(0, 7) if noise else 0)))
        bs.append(b)
        off.append(len(nid))
    return Profiles(np.array(bs), np.array(off), np.array(nid), np.array(mem), np.array(tim))


def _outcome(f, *a):
    try:
        return "ok", f(*a)
    except DagError as e:
        return "err", (e.kind, str(e))


def _same_models(a, b):
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1], b[1]), np.abs(a[1] - b[1]).max()


def _same_graph(x, y):
    for f in ("node_id", "compute_us", "memory_bytes", "edge_src", "edge_dst", "edge_bytes"):
        assert np.array_equal(getattr(x, f), getattr(y, f)), f


@pytest.mark.parametrize("batches", [(1, 2), (1, 2, 4, 8), (32, 8, 16, 8, 64), (3, 3, 5)])
def test_fit_and_estimate(est, batches):
    dp, rf = est
    rng = np.random.default_rng(len(batches))
    g = layered(7, 3000, 40)
    prof = _profiles(rng, g.node_id, batches)
    a, b = dp.fit_node_models(prof), rf.fit_node_models(prof)
    _same_models(a, b)
    ref_batch = max(batches)
    ov = [(int(g.edge_src[e]), int(g.edge_dst[e]), 0.25 + e % 3) for e in range(0, g.m, 17)]
    for target in (1, 3, 100, 12345):
        _same_graph(dp.estimate_graph(g, a, target, ref_batch, ov), rf.estimate_graph(g, b, target, ref_batch, ov))


def test_fit_large_values(est):
    dp, rf = est
    rng = np.random.default_rng(9)
    ids = np.arange(500) * 7 + 3
    prof = _profiles(rng, ids, (1 << 20, 3 << 20, 7 << 20))
    prof.memory_bytes = prof.memory_bytes * 1000003
    _same_models(dp.fit_node_models(prof), rf.fit_node_models(prof))


def test_fit_errors(est):
    dp, rf = est
    rng = np.random.default_rng(3)
    ids = np.arange(20)
    cases = [_profiles(rng, ids, (4,)), _profiles(rng, ids, (4, 4, 4))]
    p = _profiles(rng, ids, (1, 2))
    p.node_off = np.array([0, 20, 39])  # batch 2 profiles 19 nodes
    p.node_id, p.memory_bytes, p.compute_us = p.node_id[:39], p.memory_bytes[:39], p.compute_us[:39]
    cases.append(p)
    q = _profiles(rng, ids, (1, 2), shuffle=False)
    q.node_id = q.node_id.copy()
    q.node_id[25] = 99  # node 5 missing from batch 2
    cases.append(q)
    for c in cases:
        a, b = _outcome(dp.fit_node_models, c), _outcome(rf.fit_node_models, c)
        assert a[0] == b[0] == "err", (a, b)
        assert a[1] == b[1]
    g = layered(1, 50, 5)
    models = dp.fit_node_models(_profiles(rng, g.node_id[:-1], (1, 2)))
    for args in ((g, models, 0, 1), (g, models, 2, 0), (g, models, 2, 1)):
        a, b = _outcome(dp.estimate_graph, *args), _outcome(rf.estimate_graph, *args)
        assert a[0] == b[0] == "err" and a[1] == b[1], (a, b)


def test_comm_model(est):
    dp, rf = est
    rng = np.random.default_rng(4)
    for n in (2, 3, 17, 1000):
        s = [(int(rng.integers(0, 1 << 30)), float(rng.random() * 1e4)) for _ in range(n)]
        assert dp.fit_comm_model(s) == rf.fit_comm_model(s)
    for s in ([(5, 1.0)], [(5, 1.0), (5, 2.0)], [(100, 50.0), (200, 10.0)]):
        a, b = _outcome(dp.fit_comm_model, s), _outcome(rf.fit_comm_model, s)
        assert a == b


def test_deviation_report(est):
    dp, rf = est
    rng = np.random.default_rng(6)
    g = random_dag(5, 4000, 0.001)
    meas = Graph(g.node_id[::-1].copy(), rng.integers(0, 50, g.n), rng.integers(0, 5, g.n), g.edge_src, g.edge_dst,
                 g.edge_bytes)
    a, b = dp.deviation_report(g, meas), rf.deviation_report(g, meas)
    for k in ("memory", "time"):
        assert np.array_equal(a[k][0], b[k][0]) and np.array_equal(a[k][1], b[k][1])
    for k in ("zero_memory", "zero_time"):
        assert np.array_equal(a[k], b[k])
    assert a["mean_memory"] == b["mean_memory"] and a["mean_time"] == b["mean_time"]
    short = Graph(meas.node_id[:-1], meas.compute_us[:-1], meas.memory_bytes[:-1], [], [], [])
    other = Graph(np.where(meas.node_id == 7, 10 ** 9, meas.node_id), meas.compute_us, meas.memory_bytes, [], [], [])
    for m in (short, other):
        x, y = _outcome(dp.deviation_report, g, m), _outcome(rf.deviation_report, g, m)
        assert x[0] == y[0] == "err" and x[1] == y[1], (x, y)
