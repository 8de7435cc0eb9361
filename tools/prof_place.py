"""order_place + adjusting_placement of config #4's coarse graph (deep default) once, for ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2208_00184_b200 as pkg  # noqa: E402
from paper_2208_00184_b200 import synth  # noqa: E402

COMM = (0.001, 10.0)
be = pkg.device(0)
g, devs = synth.config4(len(sys.argv) < 2 or sys.argv[1] == "deep")
limit = int(min(cap for _, cap in devs) * 0.25)
coarse, cmap = be.fuse(g, COMM, 200, limit)
_, _, cc = be.compute_levels(coarse, COMM)
cseq = be.cpd_topo(coarse, cc)
be.adjusting_placement(coarse, cseq, devs, COMM)
print("placement done", flush=True)
