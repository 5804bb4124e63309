import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def lib():
    """The product library (libhepfac.so built in-tree)."""
    from paper_1704_02272_b200 import hepfac
    return hepfac.lib()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference compiled from its sources (oracle/_ref)."""
    import oracle
    r = oracle.ref_library()
    if r is None:
        pytest.skip("oracle/_ref/libhepfac_ref.so not built (needs /root/reference at build time)")
    return r


@pytest.fixture(scope="session")
def gpu(lib):
    if lib.device_count() < 1:
        pytest.fail("GPU test selected but no CUDA device is visible")
    return lib
