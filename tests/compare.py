"""Bit-exact comparison helpers shared by the parity suites."""
from __future__ import annotations

import numpy as np

from paper_2208_00184_b200._abi import DagError


def same(a, b, what=""):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    if a.size:
        bad = np.nonzero(a != b)[0] if a.ndim == 1 else np.argwhere(a != b)
        assert len(bad) == 0, f"{what}: {len(bad)} mismatches, first at {bad[0]}: {a[tuple(np.atleast_1d(bad[0]))]} vs {b[tuple(np.atleast_1d(bad[0]))]}"


def same_graph(a, b, what="graph"):
    for f in ("node_id", "compute_us", "memory_bytes", "edge_src", "edge_dst", "edge_bytes"):
        same(getattr(a, f), getattr(b, f), f"{what}.{f}")


def same_map(a, b, what="map"):
    same(a.node_cluster, b.node_cluster, f"{what}.node_cluster")
    assert a.n_clusters == b.n_clusters, f"{what}: {a.n_clusters} vs {b.n_clusters} clusters"
    oa, fa = a.member_arrays()
    ob, fb = b.member_arrays()
    same(oa, ob, f"{what}.member_off")
    same(fa, fb, f"{what}.members")
    same(a.total_compute, b.total_compute, f"{what}.total_compute")
    same(a.total_memory, b.total_memory, f"{what}.total_memory")
    same(a.breakpoints, b.breakpoints, f"{what}.breakpoints")


def same_placement(a, b, what="placement"):
    same(a.device, b.device, f"{what}.device")
    same(a.device_ids, b.device_ids, f"{what}.device_ids")
    same(a.per_device_memory, b.per_device_memory, f"{what}.per_device_memory")
    same(a.device_present, b.device_present, f"{what}.device_present")
    assert a.oom_risk == b.oom_risk, f"{what}.oom_risk"
    assert (a.decisions is None) == (b.decisions is None), f"{what}.decisions presence"
    if a.decisions is not None:
        for k in a.decisions:
            same(a.decisions[k], b.decisions[k], f"{what}.decisions.{k}")


def same_sim(a, b, what="sim"):
    assert a.makespan == b.makespan, f"{what}.makespan {a.makespan} vs {b.makespan}"
    assert a.cross_transfer_count == b.cross_transfer_count, f"{what}.cross_count"
    assert a.cross_transfer_bytes == b.cross_transfer_bytes, f"{what}.cross_bytes"
    assert a.oom_flag == b.oom_flag, f"{what}.oom"
    same(a.device_ids, b.device_ids, f"{what}.device_ids")
    same(a.peak_memory, b.peak_memory, f"{what}.peak")
    same(a.capacity, b.capacity, f"{what}.capacity")
    assert (a.trace is None) == (b.trace is None)
    if a.trace is not None:
        for k in a.trace:
            same(a.trace[k], b.trace[k], f"{what}.trace.{k}")


def same_pipeline(a, b, what="pipeline"):
    for f in ("original_nodes", "original_edges", "coarse_nodes", "coarse_edges",
              "order_makespan", "adjust_makespan"):
        assert getattr(a, f) == getattr(b, f), f"{what}.{f}: {getattr(a, f)} vs {getattr(b, f)}"
    assert a.original_ccr == b.original_ccr
    assert a.coarse_ccr == b.coarse_ccr
    same_graph(a.coarse, b.coarse, f"{what}.coarse")
    same_map(a.map, b.map, f"{what}.map")
    same(a.coarse_sequence, b.coarse_sequence, f"{what}.coarse_sequence")
    same_placement(a.coarse_order, b.coarse_order, f"{what}.coarse_order")
    same_placement(a.coarse_adjust, b.coarse_adjust, f"{what}.coarse_adjust")
    same_placement(a.order_expanded, b.order_expanded, f"{what}.order_expanded")
    same_placement(a.adjust_expanded, b.adjust_expanded, f"{what}.adjust_expanded")


def outcome(fn, *args, **kw):
    """(ok, value) or ('err', kind, message) so error behaviour compares too."""
    try:
        return ("ok", fn(*args, **kw))
    except DagError as e:
        return ("err", e.kind, str(e))


def same_outcome(a, b, cmp, what=""):
    assert a[0] == b[0], f"{what}: {a[0]} vs {b[0]} ({a[1:]} / {b[1:]})"
    if a[0] == "err":
        assert a[1] == b[1], f"{what}: kind {a[1]} vs {b[1]}"
        assert a[2] == b[2], f"{what}: message {a[2]!r} vs {b[2]!r}"
    else:
        cmp(a[1], b[1], what)
