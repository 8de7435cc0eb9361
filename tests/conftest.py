import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libdagplace_b200.so")
    config.addinivalue_line("markers", "slow: larger parity cases")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bind import oracle_backend
    return oracle_backend()


@pytest.fixture(scope="session")
def ref():
    from oracle.bind import reference_available, reference_backend
    if not reference_available():
        pytest.skip("oracle/_ref not built (reference sources unavailable)")
    return reference_backend()


@pytest.fixture(scope="session")
def gpu():
    import paper_2208_00184_b200 as pkg
    return pkg.device(0)
