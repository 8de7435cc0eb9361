"""TEST INFRASTRUCTURE ONLY — loaders for the two CPU checkers.

* ``oracle_backend()``  -> plain-C restatement, oracle/build/libdp_oracle.so (dpo_*)
* ``reference_backend()`` -> the unmodified reference sources compiled by oracle/Makefile,
  oracle/_ref/libdagplace_ref.so (dpr_*).  Absent when /root/reference was never
  available to build it; callers skip in that case.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may
import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

from paper_2208_00184_b200._abi import Backend, CommC, DevicesC, GraphC, PipelineCfgC

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libdp_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdagplace_ref.so")
REF_TESTS = os.path.join(HERE, "_ref", "ref_tests")
REF_SRC = "/root/reference/proj"

_cache = {}


def build(ref: bool = True) -> None:
    """Compile the checkers (make -C oracle [ref]); the reference only where it exists."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def oracle_backend() -> Backend:
    if "dpo" not in _cache:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        _cache["dpo"] = Backend(C.CDLL(ORACLE_SO), "dpo_", name="oracle")
    return _cache["dpo"]


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def reference_backend() -> Backend:
    if "dpr" not in _cache:
        lib = C.CDLL(REF_SO)
        be = Backend(lib, "dpr_", name="reference")
        f = lib.dpr_pipeline_replicas
        f.restype = C.c_int
        f.argtypes = [C.POINTER(GraphC), C.POINTER(DevicesC), CommC, C.POINTER(PipelineCfgC),
                      C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        be.pipeline_replicas = f
        _cache["dpr"] = be
    return _cache["dpr"]


def reference_layered(n: int, width: int, fan_lo: int = 2, fan_hi: int = 6, seed: int = 12345):
    """The SURVEY §8(d) layered recipe synthesised by oracle/_ref (dpr_gen_layered), so the
    reference arm of bench.py never maps the product library."""
    import numpy as np

    from paper_2208_00184_b200._abi import Graph
    lib = reference_backend().lib
    f = lib.dpr_gen_layered
    f.restype = C.c_int
    p64 = C.POINTER(C.c_int64)
    f.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64] + [p64] * 7
    a = [np.zeros(n, np.int64) for _ in range(3)] + [np.zeros(max(1, n * fan_hi), np.int64) for _ in range(3)]
    m = C.c_int64()
    rc = f(n, width, fan_lo, fan_hi, seed, *[x.ctypes.data_as(p64) for x in a], C.byref(m))
    if rc:
        raise RuntimeError("dpr_gen_layered failed")
    k = m.value
    return Graph(a[0], a[1], a[2], a[3][:k].copy(), a[4][:k].copy(), a[5][:k].copy())


def reference_candidates(base, D: int, first: int, count: int):
    """Config #5 candidate rows (SURVEY §8(d) family) from oracle/_ref (dpr_gen_candidates)."""
    import numpy as np
    lib = reference_backend().lib
    f = lib.dpr_gen_candidates
    f.restype = None
    u8 = C.POINTER(C.c_uint8)
    f.argtypes = [u8, C.c_int64, C.c_int32, C.c_int64, C.c_int64, u8]
    b = np.ascontiguousarray(base, dtype=np.uint8)
    out = np.zeros((count, b.size), np.uint8)
    f(b.ctypes.data_as(u8), b.size, D, first, count, out.ctypes.data_as(u8))
    return out
