"""The device-resident generation entry points that bench.py times
(dp_resident_create / dp_resident_generate / dp_resident_generate_batch /
dp_resident_fetch) against the compiled reference's evaluate_pipeline
(pipeline.cpp:27-111): identical expanded placements, identical errors — including a
cyclic graph (the generate step relies on the level pass to detect cycles) and error
ordering between graph, fusion and device-list errors."""
import ctypes as C

import numpy as np
import pytest

from cases import GEN, capacity_for, devices, invalid_graphs
from compare import outcome, same, same_outcome
from graphs import layered, random_dag

pytestmark = pytest.mark.gpu


class Resident:
    def __init__(self, gpu, g, devs, comm=GEN, fusion_range=200, frac=0.25):
        from paper_2208_00184_b200._abi import PipelineCfgC, comm_c, devices_c
        self.lib, self.g = gpu.lib, g
        self.h = C.c_void_p()
        gc, dc = g.c(), devices_c(devs)
        cfg = PipelineCfgC(fusion_range, frac, 1, 0)
        self.rc = self.lib.dp_resident_create(gpu.ctx, C.byref(gc), C.byref(dc), comm_c(comm), C.byref(cfg),
                                              C.byref(self.h))
        self.err = self.lib.dp_last_error_message().decode() if self.rc else None

    def generate(self):
        rc = self.lib.dp_resident_generate(self.h)
        return ("ok",) if rc == 0 else ("err", rc, self.lib.dp_last_error_message().decode())

    def fetch(self):
        n = self.g.n
        a, b = np.zeros(n, np.int32), np.zeros(n, np.int32)
        cn, ce = C.c_int64(), C.c_int64()
        assert self.lib.dp_resident_fetch(self.h, a.ctypes.data_as(C.POINTER(C.c_int32)),
                                          b.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(cn), C.byref(ce)) == 0
        return a, b, cn.value, ce.value

    def close(self):
        if self.h:
            self.lib.dp_resident_destroy(self.h)
            self.h = C.c_void_p()


def ref_outcome(ref, g, devs, **kw):
    o = outcome(ref.evaluate_pipeline, g, devs, GEN, **kw)
    if o[0] == "ok":
        return o
    from paper_2208_00184_b200._abi import ERROR_KINDS
    return ("err", ERROR_KINDS.index(o[1]) + 1, o[2])


@pytest.mark.parametrize("seed,n,w", [(1, 3000, 24), (2, 20000, 256), (3, 6000, 6)])
def test_resident_matches_reference(gpu, ref, seed, n, w):
    g = layered(seed, n, w)
    devs = devices(8, capacity_for(g, 8, 1.25), shuffle_seed=seed, base_id=4, stride=3)
    r = Resident(gpu, g, devs)
    try:
        assert r.rc == 0, r.err
        for _ in range(2):  # a resident regenerates identically
            assert r.generate() == ("ok",)
            a, b, cn, ce = r.fetch()
            rep = ref.evaluate_pipeline(g, devs, GEN)
            same(a, rep.order_expanded.device, "order_expanded")
            same(b, rep.adjust_expanded.device, "adjust_expanded")
            assert (cn, ce) == (rep.coarse_nodes, rep.coarse_edges)
    finally:
        r.close()


@pytest.mark.parametrize("name", ["cycle2", "cycle_tail", "dup_id", "dangling", "self_loop", "parallel", "neg_bytes", "many"])
def test_resident_invalid_graph_errors(gpu, ref, name):
    inv = invalid_graphs()
    if name not in inv:
        pytest.skip(f"no {name} case")
    g = inv[name]
    devs = devices(2, 10 ** 12)
    r = Resident(gpu, g, devs)
    try:
        assert r.rc == 0, r.err  # create only uploads; validation is part of generate
        assert r.generate() == ref_outcome(ref, g, devs)
    finally:
        r.close()


def test_resident_cycle_in_large_graph(gpu, ref):
    """A back edge deep inside a 50k-node layered graph: the resident generate path (no
    separate Kahn pass) must report the reference's cycle witness."""
    g = layered(9, 50000, 128)
    # walk 150 layers up from a node in layer 250 along in-edges, then close the path
    pred = {}
    for s_, d_ in zip(g.edge_src.tolist(), g.edge_dst.tolist()):
        pred.setdefault(d_, s_)
    end = 250 * 128 + 5
    v = end
    for _ in range(150):
        v = pred[v]
    from paper_2208_00184_b200._abi import Graph
    bad = Graph(g.node_id, g.compute_us, g.memory_bytes, np.append(g.edge_src, end), np.append(g.edge_dst, v),
                np.append(g.edge_bytes, 77))
    devs = devices(8, capacity_for(g, 8, 1.25))
    want = ref_outcome(ref, bad, devs)
    assert want[0] == "err" and want[1] == 1  # CycleDetected
    r = Resident(gpu, bad, devs)
    try:
        assert r.generate() == want
    finally:
        r.close()


def test_resident_keeps_its_own_host_copy(gpu, ref):
    """Error messages raised by a later generate name the ids of the graph as created,
    even after the caller overwrote its arrays."""
    g = invalid_graphs()["dangling"]
    devs = devices(2, 10 ** 12)
    want = ref_outcome(ref, g, devs)
    from paper_2208_00184_b200._abi import Graph
    mine = Graph(g.node_id.copy(), g.compute_us.copy(), g.memory_bytes.copy(), g.edge_src.copy(),
                 g.edge_dst.copy(), g.edge_bytes.copy())
    r = Resident(gpu, mine, devs)
    try:
        for a in (mine.node_id, mine.edge_src, mine.edge_dst):
            a[...] = -12345
        assert r.generate() == want
    finally:
        r.close()


def error_order_cases():
    good = layered(5, 2000, 16)
    bad_graph = invalid_graphs()["dup_id"]
    cap = capacity_for(good, 4, 1.25)
    dup_dev = [(1, cap), (1, cap), (2, cap)]
    zero_dev = [(0, cap), (1, 0)]
    return {
        "graph_and_devices_invalid": (bad_graph, dup_dev, {}),
        "dup_devices": (good, dup_dev, {}),
        "zero_capacity_device": (good, zero_dev, {}),  # limit = max(1, 0) -> NodeExceedsClusterLimit
        "fusion_range_zero": (good, devices(4, cap), {"fusion_range": 0}),
        "fusion_range_zero_and_bad_devices": (good, dup_dev, {"fusion_range": 0}),
        "empty_devices": (good, [], {}),
    }


@pytest.mark.parametrize("name", sorted(error_order_cases()))
def test_pipeline_error_order(gpu, ref, oracle, name):
    g, devs, kw = error_order_cases()[name]
    want = outcome(ref.evaluate_pipeline, g, devs, GEN, **kw)
    assert want[0] == "err"
    same_outcome(outcome(gpu.evaluate_pipeline, g, devs, GEN, **kw), want, None, name)
    same_outcome(outcome(oracle.evaluate_pipeline, g, devs, GEN, **kw), want, None, name)
    if devs:
        r = Resident(gpu, g, devs, fusion_range=kw.get("fusion_range", 200))
        try:
            assert r.rc == 0, r.err
            assert r.generate() == ref_outcome(ref, g, devs, **kw)
        finally:
            r.close()


def test_resident_many_devices(gpu, ref):
    g = random_dag(4, 3000, 0.002)
    devs = devices(24, capacity_for(g, 24, 1.25))
    r = Resident(gpu, g, devs)
    try:
        assert r.generate() == ("ok",)
        a, b, _, _ = r.fetch()
        rep = ref.evaluate_pipeline(g, devs, GEN)
        same(a, rep.order_expanded.device, "order")
        same(b, rep.adjust_expanded.device, "adjust")
    finally:
        r.close()
