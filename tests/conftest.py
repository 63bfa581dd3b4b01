import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size (BASELINE.json) configs")


@pytest.fixture(scope="session", autouse=True)
def _native_libs():
    from tools import build
    build.build_gen()
    build.build_oracle()
    yield


@pytest.fixture(scope="session")
def bq():
    """The CUDA path's Python binding (builds libbq.so if stale)."""
    from tools import build
    build.build_bq()
    import paper_1604_06697_b200 as pkg
    return pkg
