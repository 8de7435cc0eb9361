"""The tree peel (cpd_topo) of config #4's graph once per variant, with DP_DEBUG_FIXPOINT phase
clocks: python tools/prof_tree.py [deep|wide]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("DP_DEBUG_FIXPOINT", "1")

import paper_2208_00184_b200 as pkg  # noqa: E402
from paper_2208_00184_b200 import synth  # noqa: E402

COMM = (0.001, 10.0)
be = pkg.device(0)
g, _ = synth.config4(len(sys.argv) < 2 or sys.argv[1] == "deep")
_, _, c = be.compute_levels(g, COMM)
for _ in range(3):
    be.cpd_topo(g, c)
print("tree done", flush=True)
