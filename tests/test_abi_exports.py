"""CPU-side checks of the C-ABI boundary: the library loads without a GPU, exports every
symbol include/dagplace_b200.h declares, and fails loudly (no CPU fallback) when no
CUDA device is present."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2208_00184_b200", "libdagplace_b200.so")
HDR = os.path.join(ROOT, "include", "dagplace_b200.h")


def header_functions():
    text = open(HDR).read()
    return sorted(n for n in set(re.findall(r"\b(dp_[a-z0-9_]+)\s*\(", text)) if not n.endswith("_t"))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        pytest.skip("libdagplace_b200.so not built")
    return ctypes.CDLL(LIB)


def test_every_header_symbol_exported(lib):
    from paper_2208_00184_b200._native import HEADER_SYMBOLS
    names = header_functions()
    assert set(names) == set(HEADER_SYMBOLS), set(names) ^ set(HEADER_SYMBOLS)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2208_00184_b200 as pkg
    with pytest.raises(pkg.DagError) as e:
        pkg.device(0)
    assert "no CPU fallback" in str(e.value)


def test_generator_matches_recipe(lib):
    """dp_gen_layered (host synthesis) reproduces the survey's common recipe shape."""
    import numpy as np
    from paper_2208_00184_b200 import synth
    g = synth.layered(5000, 32, 2, 6, 12345)
    assert g.n == 5000 and 2 * (5000 - 32) <= g.m <= 6 * (5000 - 32)
    assert np.all(np.diff(g.edge_src) >= 0)
    assert g.compute_us.min() >= 100 and g.compute_us.max() <= 900
    g2 = synth.layered(5000, 32, 2, 6, 12345)
    assert np.array_equal(g.edge_bytes, g2.edge_bytes)
