"""Per-stage device timings of the sequential kernels on the 1M-op config #4 graph
(diagnostics for optimisation; run on the GPU box).  Uses the context's stage timing
(CUDA events on the launching stream around each kernel stage)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2208_00184_b200 as pkg  # noqa: E402
from paper_2208_00184_b200 import synth  # noqa: E402
from paper_2208_00184_b200._native import stage_times  # noqa: E402

COMM = (0.001, 10.0)


def timed(be, fn, *args):
    lib = pkg.library()
    lib.dp_ctx_enable_stage_timing(be.ctx, 1)
    t = time.perf_counter()
    out = fn(*args)
    wall = time.perf_counter() - t
    st = stage_times(lib, be.ctx)
    lib.dp_ctx_enable_stage_timing(be.ctx, 0)
    return out, wall, st


def main():
    variant = sys.argv[1] if len(sys.argv) > 1 else "deep"
    be = pkg.device(0)
    g, devs = synth.config4(variant == "deep")
    (t, b, c), wall, st = timed(be, be.compute_levels, g, COMM)
    print(f"compute_levels wall {wall:.3f}s", [(n, round(ms, 3)) for n, ms, _ in st])
    seq, wall, st = timed(be, be.cpd_topo, g, c)
    print(f"cpd_topo wall {wall:.3f}s", [(n, round(ms, 3)) for n, ms, _ in st])
    seq2, wall, st = timed(be, be.dfs_topo, g)
    print(f"dfs_topo wall {wall:.3f}s", [(n, round(ms, 3)) for n, ms, _ in st])
    limit = int(min(cap for _, cap in devs) * 0.25)
    m, wall, st = timed(be, be.optimal_breakpoints, g, seq, COMM, 200, limit)
    print(f"optimal_breakpoints wall {wall:.3f}s clusters={m.n_clusters}", [(n, round(ms, 3)) for n, ms, _ in st])
    (coarse, cmap), wall, st = timed(be, be.fuse, g, COMM, 200, limit)
    print(f"fuse wall {wall:.3f}s coarse={coarse.n}", [(n, round(ms, 3)) for n, ms, _ in st])
    _, _, cc = be.compute_levels(coarse, COMM)
    cseq = be.cpd_topo(coarse, cc)
    p, wall, st = timed(be, be.adjusting_placement, coarse, cseq, devs, COMM)
    print(f"adjusting wall {wall:.3f}s", [(n, round(ms, 3)) for n, ms, _ in st])
    p, wall, st = timed(be, be.order_place, coarse, cseq, devs)
    print(f"order_place wall {wall:.3f}s", [(n, round(ms, 3)) for n, ms, _ in st])
    np.save("/tmp/seq.npy", seq)


if __name__ == "__main__":
    main()
