"""One fuse() of config #4 (deep by default) for ncu captures of the DP / tree-peel kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2208_00184_b200 as pkg  # noqa: E402
from paper_2208_00184_b200 import synth  # noqa: E402

be = pkg.device(0)
g, devs = synth.config4(len(sys.argv) < 2 or sys.argv[1] == "deep")
limit = int(min(cap for _, cap in devs) * 0.25)
be.fuse(g, (0.001, 10.0), 200, limit)
print("fuse done", flush=True)
