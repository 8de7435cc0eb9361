"""Level-kernel probe (diagnostics; run on the GPU box): compute_levels on the config #4
deep and wide graphs (and the coarse graph of each) under several dataflow switch settings,
reporting the 'levels' stage time (CUDA events on the launching stream; min / median of
`reps`), the achieved algorithmic GB/s (40 B/edge + 48 B/node, DESIGN 3.2) and whether the
levels equal those of the default setting bit for bit."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2208_00184_b200 as pkg  # noqa: E402
from paper_2208_00184_b200 import synth  # noqa: E402
from paper_2208_00184_b200._native import stage_times  # noqa: E402

COMM = (0.001, 10.0)
SETTINGS = [
    {},
    {"DP_FLOW_GRAIN": "1"},
    {"DP_FLOW_GRAIN": "2"},
    {"DP_FLOW_GRAIN": "8"},
    {"DP_FLOW_WARPS": "4"},
    {"DP_FLOW_WARPS": "16"},
    {"DP_FLOW_WARPS": "4", "DP_FLOW_GRAIN": "8"},
    {"DP_FLOW_WARPS": "16", "DP_FLOW_GRAIN": "8"},
    {"DP_FLOW_GRAIN": "2", "DP_FLOW_AHEAD": "64"},
]
KEYS = ("DP_FLOW_AHEAD", "DP_FLOW_SLEEP", "DP_FLOW_WARPS", "DP_FLOW_POLL_ALL", "DP_FLOW_GRAIN")
KEYS = ("DP_FLOW_AHEAD", "DP_FLOW_SLEEP", "DP_FLOW_WARPS", "DP_FLOW_POLL_ALL")
KEYS = ("DP_FLOW_AHEAD", "DP_FLOW_SLEEP", "DP_FLOW_WARPS")


def levels_ms(be, g, reps):
    lib = pkg.library()
    ms, out = [], None
    for _ in range(reps):
        lib.dp_ctx_enable_stage_timing(be.ctx, 1)
        out = be.compute_levels(g, COMM)
        st = stage_times(lib, be.ctx)
        lib.dp_ctx_enable_stage_timing(be.ctx, 0)
        ms.append(sum(t for name, t, _ in st if name == "levels"))
    return sorted(ms), out


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 7
    env_only = len(sys.argv) > 2 and sys.argv[2] == "env"  # one run under the caller's environment
    settings = [{}] if env_only else SETTINGS
    be = pkg.device(0)
    for variant in ("wide", "deep"):
        g, _ = synth.config4(variant == "deep")
        bytes_ = 40.0 * g.m + 48.0 * g.n
        base = None
        for s in settings:
            if not env_only:
                for k in KEYS:
                    os.environ.pop(k, None)
                os.environ.update(s)
            ms, (t, b, c) = levels_ms(be, g, reps)
            if base is None:
                base = (t, b, c)
            same = all(np.array_equal(x, y) for x, y in zip((t, b, c), base))
            print(f"{variant} {s or 'default'}: min {ms[0]:.4f} ms median {ms[len(ms) // 2]:.4f} ms "
                  f"{bytes_ / ms[0] / 1e6:.1f} GB/s same={same}", flush=True)


if __name__ == "__main__":
    main()
