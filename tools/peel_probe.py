"""The CPD peel alone on config #4 (k_peel2 through dp_topo_order), for timing and ncu
source-level stall sampling without the DP warps of the streamed kernel:

    python tools/peel_probe.py [deep|wide] [reps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2208_00184_b200 as pkg  # noqa: E402
from paper_2208_00184_b200 import synth  # noqa: E402

variant = sys.argv[1] if len(sys.argv) > 1 else "deep"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
be = pkg.device(0)
g, _ = synth.config4(variant == "deep")
_, _, cp = be.compute_levels(g, (0.001, 10.0))
for i in range(reps):
    t = time.perf_counter()
    seq = be.cpd_topo(g, cp)
    print(f"cpd_topo {variant}: {1e3 * (time.perf_counter() - t):.1f} ms (host wall, incl. upload + index)", flush=True)
