"""B200-native graph-analysis / placement-evaluation path of Celeritas (dagplace).

The compute lives in libdagplace_b200.so (hand-written sm_100a CUDA behind the C-ABI of
include/dagplace_b200.h).  This package is the Python host surface over that ABI; it
mirrors the reference's C++ API names (compute_levels, cpd_topo, fuse, order_place,
adjusting_placement, simulate, evaluate_pipeline, ...).  There is no CPU fallback:
`device()` raises if the extension or a CUDA device is missing.
"""
from __future__ import annotations

import ctypes as C
import os

from ._abi import (DagError, Graph, Backend, TOPO_CPD, TOPO_DFS, TOPO_M, UNPLACED, NEVER,  # noqa: F401
                   ClusterMap, Placement, SimReport, PipelineReport)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdagplace_b200.so")

_lib = None
_backends = {}


def library() -> C.CDLL:
    """Load libdagplace_b200.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libdagplace_b200.so missing at {LIB_PATH}; run __graft_entry__.build()")
        _lib = C.CDLL(LIB_PATH)
        from . import _native  # noqa: F401  (declares ctx/resident/gen signatures)
        _native.declare(_lib)
    return _lib


def device(index: int = 0, stream: int | None = None) -> Backend:
    """Backend bound to a dp_ctx_t on CUDA device `index` (optionally a cudaStream_t)."""
    key = (index, stream)
    if key not in _backends:
        lib = library()
        ctx = C.c_void_p()
        rc = lib.dp_ctx_create(index, C.c_void_p(stream) if stream else None, C.byref(ctx))
        if rc != 0:
            raise DagError(rc, lib.dp_last_error_message().decode())
        _backends[key] = Backend(lib, "dp_", ctx=ctx, name=f"cuda:{index}")
    return _backends[key]
