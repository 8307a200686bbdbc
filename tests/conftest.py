import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


def gpu_count() -> int:
    import ctypes as C

    from paper_1709_00700_b200 import _native
    n = C.c_int32(0)
    _native.b200().hawk_b200_device_count(C.byref(n))
    return n.value


@pytest.fixture(scope="session")
def engine():
    if gpu_count() < 1:
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_1709_00700_b200 import Engine
    e = Engine(0)
    yield e
    e.close()


@pytest.fixture
def planner():
    """Planning-only engine (no GPU): catalog, passes, variant space, lowering."""
    from paper_1709_00700_b200 import Engine
    e = Engine(-1)
    yield e
    e.close()
