import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_lib import RefLib, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built (reference sources absent on this host)")
    return RefLib()


@pytest.fixture(scope="session")
def bode():
    import paper_1611_02274_b200 as B
    B.lib()
    return B


@pytest.fixture(scope="session")
def gpu(bode):
    """The product library on a real device; fails (never skips) when absent."""
    n = bode.lib().bode_device_count()
    assert n >= 1, "gpu-marked test needs a CUDA device: no CPU fallback exists"
    return bode
