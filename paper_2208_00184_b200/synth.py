"""Deterministic synthetic inputs for benches and tests (SURVEY §8(d) recipes), generated
by the library's host-side generator dp_gen_layered."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._abi import Graph


def _lib():
    from . import library
    return library()


def layered(n: int, width: int, fan_lo: int = 2, fan_hi: int = 6, seed: int = 12345) -> Graph:
    lib = _lib()
    cap = max(1, n * fan_hi)
    a = [np.zeros(n, np.int64) for _ in range(3)] + [np.zeros(cap, np.int64) for _ in range(3)]
    m = C.c_int64()
    p = lambda x: x.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731
    rc = lib.dp_gen_layered(n, width, fan_lo, fan_hi, seed, *[p(x) for x in a], C.byref(m))
    if rc:
        raise RuntimeError(lib.dp_last_error_message().decode())
    k = m.value
    return Graph(a[0], a[1], a[2], a[3][:k].copy(), a[4][:k].copy(), a[5][:k].copy())


def _run(fn, n, cap_edges, *lead):
    lib = _lib()
    a = [np.zeros(n, np.int64) for _ in range(3)] + [np.zeros(cap_edges, np.int64) for _ in range(3)]
    m = C.c_int64()
    p = lambda x: x.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731
    rc = getattr(lib, fn)(*lead, *[p(x) for x in a], C.byref(m))
    if rc:
        raise RuntimeError(lib.dp_last_error_message().decode())
    k = m.value
    return Graph(a[0], a[1], a[2], a[3][:k].copy(), a[4][:k].copy(), a[5][:k].copy())


def gnmt(chains: int = 8, T: int = 6250, seed: int = 2) -> Graph:
    """Config #2: GNMT-like chains (dp_gen_gnmt)."""
    return _run("dp_gen_gnmt", chains * T, chains * T * 3, chains, T, seed)


def bert(n: int = 200_000, width: int = 512, skip: int = 16, seed: int = 3) -> Graph:
    """Config #3: BERT-like layered + skip edges (dp_gen_bert)."""
    return _run("dp_gen_bert", n, n * 7, n, width, skip, seed)


def capacity_125(g: Graph, d: int) -> int:
    """#4/#5 device capacity: total/D + total/(4D) in integer arithmetic."""
    total = int(g.memory_bytes.sum())
    return total // d + total // (4 * d)


def config4(deep: bool = True):
    """Config #4: 1M ops, fan-in 2..6, seed 12345, 8 devices; deep W=1024 or wide W=65,536."""
    g = layered(1_000_000, 1024 if deep else 65536, 2, 6, 12345)
    cap = capacity_125(g, 8)
    return g, [(d, cap) for d in range(8)]


def config5_graph():
    """Config #5 graph: 100k ops, W=256, fan-in 2..6, seed 12345, 8 devices."""
    g = layered(100_000, 256, 2, 6, 12345)
    cap = capacity_125(g, 8)
    return g, [(d, cap) for d in range(8)]


def candidates(base_dev_pos: np.ndarray, D: int, first: int, count: int) -> np.ndarray:
    """Config #5 candidate family rows first..first+count-1 (dp_gen_candidates)."""
    lib = _lib()
    base = np.ascontiguousarray(base_dev_pos, dtype=np.uint8)
    out = np.zeros((count, base.size), np.uint8)
    u8 = C.POINTER(C.c_uint8)
    rc = lib.dp_gen_candidates(base.ctypes.data_as(u8), base.size, D, first, count, out.ctypes.data_as(u8))
    if rc:
        raise RuntimeError(lib.dp_last_error_message().decode())
    return out
