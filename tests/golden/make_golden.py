"""Generate golden digests of the BASELINE configs by running the UNMODIFIED reference
(oracle/_ref/libdagplace_ref.so, compiled from /root/reference/proj/src) — run here,
where /root/reference exists:

    python tests/golden/make_golden.py [--configs 1,2,3,4d,4w,5]

Writes tests/golden/configs.json: per config the graph digest, coarse sizes, and SHA-256
digests of every pipeline output (coarse graph, cluster map, coarse sequence, both
coarse placements + decision log, both expanded placements) plus both makespans.  The
GPU tests recompute the same digests from libdagplace_b200 and require equality.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from golden_configs import CONFIGS, build_config  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def device_digest(dev) -> str:
    """Digest of an expanded placement's device ids by node index (int32): what
    dp_resident_fetch returns, so bench.py can check its own timed outputs."""
    return digest(np.ascontiguousarray(dev, dtype=np.int32))


def pipeline_digests(rep) -> dict:
    off, flat = rep.map.member_arrays()
    d = {
        "coarse_nodes": rep.coarse_nodes, "coarse_edges": rep.coarse_edges,
        "coarse": digest(rep.coarse.compute_us, rep.coarse.memory_bytes, rep.coarse.edge_src, rep.coarse.edge_dst,
                         rep.coarse.edge_bytes),
        "map": digest(rep.map.node_cluster, off, flat, rep.map.total_compute, rep.map.total_memory,
                      rep.map.breakpoints),
        "coarse_sequence": digest(rep.coarse_sequence),
        "coarse_order": digest(rep.coarse_order.device, rep.coarse_order.per_device_memory,
                               np.array([rep.coarse_order.oom_risk])),
        "coarse_adjust": digest(rep.coarse_adjust.device, rep.coarse_adjust.per_device_memory,
                                np.array([rep.coarse_adjust.oom_risk])),
        "decisions": digest(*[rep.coarse_adjust.decisions[k] for k in sorted(rep.coarse_adjust.decisions)]),
        "order_expanded": digest(rep.order_expanded.device, rep.order_expanded.per_device_memory,
                                 rep.order_expanded.device_present),
        "adjust_expanded": digest(rep.adjust_expanded.device, rep.adjust_expanded.per_device_memory,
                                  rep.adjust_expanded.device_present),
        "order_device": device_digest(rep.order_expanded.device),
        "adjust_device": device_digest(rep.adjust_expanded.device),
        "order_makespan": rep.order_makespan, "adjust_makespan": rep.adjust_makespan,
        "original_ccr": rep.original_ccr, "coarse_ccr": rep.coarse_ccr,
    }
    return d


def graph_digest(g) -> str:
    return digest(g.node_id, g.compute_us, g.memory_bytes, g.edge_src, g.edge_dst, g.edge_bytes)


CAND_PREFIX = 512


def candidate_prefix(ref, threads: int):
    """Config #5: makespans of candidates 0..CAND_PREFIX-1 of the family
    around the reference's adjusting placement, simulated by the reference (a loop of
    simulate(), simulator.cpp:56-252), and the first strict minimum (:292-294)."""
    from golden_configs import config5_candidates
    g, devs, comm, rep, cand = config5_candidates(ref, 0, CAND_PREFIX)
    t = time.time()
    ms, am = ref.simulate_candidates(g, rep.map.node_cluster, rep.coarse_nodes, cand, devs, comm, threads)
    dt = time.time() - t
    return {"first": 0, "count": CAND_PREFIX, "makespans": [int(x) for x in ms], "argmin": int(am),
            "base_digest": digest(cand[0]), "rows_digest": digest(cand), "reference_seconds": round(dt, 2),
            "reference_threads": threads}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default=",".join(CONFIGS))
    ap.add_argument("--candidates", action="store_true", help="(re)write tests/golden/candidates5.json")
    args = ap.parse_args()
    from oracle.bind import reference_backend
    ref = reference_backend()
    if args.candidates:
        c = candidate_prefix(ref, os.cpu_count() or 1)
        json.dump(c, open(os.path.join(HERE, "candidates5.json"), "w"), indent=0)
        print("candidates", c["count"], "argmin", c["argmin"], c["makespans"][c["argmin"]], c["reference_seconds"], "s")
        return
    path = os.path.join(HERE, "configs.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for name in args.configs.split(","):
        g, devs, comm = build_config(name)
        t = time.time()
        rep = ref.evaluate_pipeline(g, devs, comm, simulate=True)
        dt = time.time() - t
        entry = {"graph": graph_digest(g), "n": g.n, "m": g.m, "devices": devs, "comm": comm,
                 "reference_seconds": round(dt, 2), **pipeline_digests(rep)}
        out[name] = entry
        print(name, g.n, g.m, rep.coarse_nodes, rep.order_makespan, rep.adjust_makespan, f"{dt:.1f}s", flush=True)
        json.dump(out, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
