import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session", autouse=True)
def _built_libraries():
    """Both the oracle (test infrastructure) and the product library are
    built in-tree before any test runs (seconds when up to date)."""
    from oracle import oracle as orc
    import paper_2107_01745_b200 as so

    orc.build()
    so.build()
    yield


@pytest.fixture(scope="session")
def gpu():
    import paper_2107_01745_b200 as so

    if so.device_count() < 1:
        pytest.fail("no sm_100 device visible: GPU tests must run on a B200 box")
    return 0
