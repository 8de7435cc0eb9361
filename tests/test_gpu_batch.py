"""dp_pipeline_batch / dp_resident_generate_batch: independent graphs evaluated in one call
(their peel + DP cores share one cooperative launch, 4 graphs per launch) must give, graph
by graph, exactly the reference's evaluate_pipeline (oracle/_ref); a failing graph fails the
call with that graph's error kind and message."""
import numpy as np
import pytest

from compare import outcome, same_pipeline
from graphs import layered, random_dag, shuffled, with_groups
from cases import GEN, capacity_for, devices

pytestmark = pytest.mark.gpu


def _batch_graphs():
    gs = [layered(40 + s, 2000 + 700 * s, 30 + 10 * s) for s in range(5)]
    gs.append(shuffled(layered(50, 4000, 64), 1, relabel=True))   # Kahn levels path
    for s in range(3):  # co-location contraction (some group draws are cyclic: filtered below)
        gs.append(with_groups(layered(51 + s, 3000, 40), s, 20, 0.05))
    gs.append(random_dag(55, 1500, 0.004))
    gs.append(layered(53, 1, 1))                                   # single node
    return gs


def test_pipeline_batch_matches_reference(gpu, ref):
    gs = _batch_graphs()
    cap = max(capacity_for(g, 4, 1.25) for g in gs)
    devs = devices(4, cap)
    gs = [g for g in gs if outcome(ref.evaluate_pipeline, g, devs, GEN)[0] == "ok"]
    assert len(gs) >= 7
    got = gpu.evaluate_pipeline_batch(gs, devs, GEN)
    assert len(got) == len(gs)
    for i, (g, r) in enumerate(zip(gs, got)):
        same_pipeline(r, ref.evaluate_pipeline(g, devs, GEN), f"batch[{i}]")


def test_pipeline_batch_error_and_empty(gpu, ref):
    good = layered(60, 3000, 40)
    bad = layered(61, 2000, 40)
    bad.memory_bytes = bad.memory_bytes.copy()
    bad.memory_bytes[17] = 10 ** 15  # exceeds the cluster limit: NodeExceedsClusterLimit
    devs = devices(4, capacity_for(good, 4, 1.25))
    a = outcome(gpu.evaluate_pipeline_batch, [good, bad, good], devs, GEN)
    b = outcome(ref.evaluate_pipeline, bad, devs, GEN)
    assert a[0] == b[0] == "err" and a[1:] == b[1:], (a[:1], b[:1])
    assert gpu.evaluate_pipeline_batch([], devs, GEN) == []
    # the context stays usable after a failed batch
    same_pipeline(gpu.evaluate_pipeline_batch([good], devs, GEN)[0], ref.evaluate_pipeline(good, devs, GEN))


def test_resident_generate_batch_matches_single(gpu):
    """dp_resident_generate_batch (the throughput path of bench.py) against one
    dp_resident_generate per graph: identical expanded placements and coarse sizes."""
    import ctypes as C
    from paper_2208_00184_b200._abi import PipelineCfgC, comm_c, devices_c
    lib = gpu.lib
    gs = [layered(70 + s, 5000 + 1000 * s, 50 + 20 * s) for s in range(5)]
    devs = devices(8, max(capacity_for(g, 8, 1.25) for g in gs))
    cfg = PipelineCfgC(200, 0.25, 1, 0)
    dc = devices_c(devs)

    def create(g):
        h = C.c_void_p()
        gc = g.c()
        assert lib.dp_resident_create(gpu.ctx, C.byref(gc), C.byref(dc), comm_c(GEN), C.byref(cfg), C.byref(h)) == 0
        return h.value

    def fetch(h, g):
        a, b = np.zeros(g.n, np.int32), np.zeros(g.n, np.int32)
        cn, ce = C.c_int64(), C.c_int64()
        assert lib.dp_resident_fetch(C.c_void_p(h), a.ctypes.data_as(C.POINTER(C.c_int32)),
                                     b.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(cn), C.byref(ce)) == 0
        return a, b, cn.value, ce.value

    single, batch = [create(g) for g in gs], [create(g) for g in gs]
    try:
        for h in single:
            assert lib.dp_resident_generate(C.c_void_p(h)) == 0
        arr = (C.c_void_p * len(batch))(*batch)
        assert lib.dp_resident_generate_batch(arr, len(batch)) == 0
        for g, h1, h2 in zip(gs, single, batch):
            x, y = fetch(h1, g), fetch(h2, g)
            assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1]) and x[2:] == y[2:]
    finally:
        for h in single + batch:
            lib.dp_resident_destroy(C.c_void_p(h))


def test_pipeline_batch_chunks_beyond_launch_width(gpu, ref):
    """12 graphs in one call: the per-launch argument batches (8 graphs for the peel + DP,
    coarse sweep, coarse peel and placement launches) are split across two launches."""
    gs = [layered(80 + s, 800 + 150 * s, 16 + 4 * (s % 5)) for s in range(12)]
    devs = devices(4, max(capacity_for(g, 4, 1.25) for g in gs))
    got = gpu.evaluate_pipeline_batch(gs, devs, GEN)
    for i, (g, r) in enumerate(zip(gs, got)):
        same_pipeline(r, ref.evaluate_pipeline(g, devs, GEN), f"batch12[{i}]")


def test_batch_errors_in_order(gpu, ref):
    """Validation and the generation windows are batched (one host sync per phase for the
    whole call), yet the call fails with the error of the FIRST failing graph in call
    order, as a loop of single calls would: a window-stage failure (NodeExceedsClusterLimit
    in fuse) in graph 1 wins over a validation failure (CycleDetected) in graph 2, and vice
    versa when the order is swapped."""
    from paper_2208_00184_b200._abi import Graph
    good = layered(62, 3000, 40)
    heavy = layered(63, 2000, 40)
    heavy.memory_bytes = heavy.memory_bytes.copy()
    heavy.memory_bytes[5] = 10 ** 15
    cyc = Graph(np.array([1, 2, 3]), np.array([5, 5, 5]), np.array([1, 1, 1]), np.array([1, 2, 3]),
                np.array([2, 3, 1]), np.array([10, 10, 10]))
    devs = devices(4, capacity_for(good, 4, 1.25))
    for order, first in (([good, heavy, cyc], heavy), ([good, cyc, heavy], cyc), ([cyc, good, heavy], cyc)):
        a = outcome(gpu.evaluate_pipeline_batch, order, devs, GEN)
        b = outcome(ref.evaluate_pipeline, first, devs, GEN)
        assert a[0] == b[0] == "err" and a[1:] == b[1:], (a, b)
    same_pipeline(gpu.evaluate_pipeline_batch([good], devs, GEN)[0], ref.evaluate_pipeline(good, devs, GEN))
