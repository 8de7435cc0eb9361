"""Backend-agnostic parity drivers: run the same reference-API call on two backends
and require identical results (bit-exact) or identical errors (kind + message)."""
from __future__ import annotations

import numpy as np

from cases import GEN, HALF, ODD, UNIT, capacity_for, devices
from compare import (outcome, same, same_graph, same_map, same_outcome, same_pipeline,
                     same_placement, same_sim)

COMMS = [UNIT, GEN, HALF, ODD]


def _eq(a, b, what):
    if isinstance(a, tuple):
        assert len(a) == len(b)
        for i, (x, y) in enumerate(zip(a, b)):
            _eq(x, y, f"{what}[{i}]")
    elif isinstance(a, np.ndarray):
        same(a, b, what)
    elif isinstance(a, list):
        assert len(a) == len(b), f"{what}: len {len(a)} vs {len(b)}"
        for i, (x, y) in enumerate(zip(a, b)):
            _eq(x, y, f"{what}[{i}]")
    elif hasattr(a, "__dataclass_fields__"):
        for k in a.__dataclass_fields__:
            _eq(getattr(a, k), getattr(b, k), f"{what}.{k}")
    elif isinstance(a, dict):
        assert a.keys() == b.keys()
        for k in a:
            _eq(a[k], b[k], f"{what}.{k}")
    else:
        assert a == b, f"{what}: {a!r} vs {b!r}"


def check_core(a, b, g, name=""):
    """validate / require_valid / ccr / index / levels / orders on one graph."""
    _eq(a.validate(g), b.validate(g), f"{name} validate")
    same_outcome(outcome(a.require_valid, g), outcome(b.require_valid, g), _eq, f"{name} require_valid")
    for comm in COMMS:
        same_outcome(outcome(a.ccr, g, comm), outcome(b.ccr, g, comm), _eq, f"{name} ccr{comm}")
        same_outcome(outcome(a.compute_levels, g, comm), outcome(b.compute_levels, g, comm), _eq,
                     f"{name} levels{comm}")
    ok = outcome(a.require_valid, g)[0] == "ok"
    if ok:
        _eq(a.graph_index(g), b.graph_index(g), f"{name} index")
        same_outcome(outcome(a.m_topo, g), outcome(b.m_topo, g), _eq, f"{name} m_topo")
        same_outcome(outcome(a.dfs_topo, g), outcome(b.dfs_topo, g), _eq, f"{name} dfs_topo")
        for comm in (UNIT, GEN):
            _, _, cp = b.compute_levels(g, comm)
            sa = outcome(a.cpd_topo, g, cp)
            sb = outcome(b.cpd_topo, g, cp)
            same_outcome(sa, sb, _eq, f"{name} cpd_topo{comm}")
            if sa[0] == "ok":
                assert a.is_valid_topo_order(g, sa[1]) and b.is_valid_topo_order(g, sa[1])
    else:
        for pol in (0, 1):
            same_outcome(outcome(a.topo_order, g, pol), outcome(b.topo_order, g, pol), _eq,
                         f"{name} topo{pol}")


def check_fusion(a, b, g, name="", ranges=(1, 3, 200), fracs=(0.05, 0.3, 10.0)):
    """optimal_breakpoints / build_coarse_graph / contract / fuse across limits."""
    if outcome(b.require_valid, g)[0] != "ok":
        return
    _, _, cp = b.compute_levels(g, GEN)
    seq = b.cpd_topo(g, cp)
    total = int(g.memory_bytes.sum()) if g.n else 1
    for r in ranges:
        for f in fracs:
            limit = max(1, int(total * f))
            for comm in (UNIT, GEN):
                ma = outcome(a.optimal_breakpoints, g, seq, comm, r, limit)
                mb = outcome(b.optimal_breakpoints, g, seq, comm, r, limit)
                same_outcome(ma, mb, same_map, f"{name} breakpoints r{r} f{f} {comm}")
                if mb[0] == "ok" and comm == GEN:
                    m = mb[1]
                    ca = outcome(a.build_coarse_graph, g, seq, g.node_id, m.node_cluster, m.members)
                    cb = outcome(b.build_coarse_graph, g, seq, g.node_id, m.node_cluster, m.members)
                    same_outcome(ca, cb, same_graph, f"{name} coarse r{r} f{f}")
            fa = outcome(a.fuse, g, GEN, r, limit)
            fb = outcome(b.fuse, g, GEN, r, limit)
            same_outcome(fa, fb, lambda x, y, w: (same_graph(x[0], y[0], w), same_map(x[1], y[1], w)),
                         f"{name} fuse r{r} f{f}")
    same_outcome(outcome(a.contract_colocation_groups, g), outcome(b.contract_colocation_groups, g),
                 _eq, f"{name} contract")


def check_placement(a, b, g, name=""):
    if outcome(b.require_valid, g)[0] != "ok" or g.n == 0:
        return
    _, _, cp = b.compute_levels(g, GEN)
    seq = b.cpd_topo(g, cp)
    for d, factor, sh in ((1, 2.0, None), (3, 1.25, 7), (4, 0.6, None), (8, 0.2, 3)):
        devs = devices(d, capacity_for(g, d, factor), shuffle_seed=sh, base_id=2, stride=3)
        same_outcome(outcome(a.order_place, g, seq, devs), outcome(b.order_place, g, seq, devs),
                     same_placement, f"{name} order_place d{d}")
        for comm in (UNIT, GEN, HALF):
            same_outcome(outcome(a.adjusting_placement, g, seq, devs, comm),
                         outcome(b.adjusting_placement, g, seq, devs, comm),
                         same_placement, f"{name} adjust d{d} {comm}")


def check_simulate(a, b, g, name="", seeds=(0, 1, 2)):
    if outcome(b.require_valid, g)[0] != "ok" or g.n == 0:
        return
    for s in seeds:
        rng = np.random.default_rng(s)
        d = [1, 2, 3, 5][s % 4]
        devs = devices(d, capacity_for(g, d, 0.9), shuffle_seed=s, base_id=1, stride=2)
        ids = np.array(sorted(x[0] for x in devs), np.int32)
        place = ids[rng.integers(0, d, g.n)]
        for comm in (UNIT, GEN):
            same_outcome(outcome(a.simulate, g, place, devs, comm, True),
                         outcome(b.simulate, g, place, devs, comm, True), same_sim,
                         f"{name} simulate s{s} {comm}")


def check_pipeline(a, b, g, name="", d=4):
    if outcome(b.require_valid, g)[0] != "ok" or g.n == 0:
        return
    devs = devices(d, capacity_for(g, d, 1.25))
    same_outcome(outcome(a.evaluate_pipeline, g, devs, GEN), outcome(b.evaluate_pipeline, g, devs, GEN),
                 same_pipeline, f"{name} pipeline")
