import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running (minutes)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def lib():
    """The product binding; builds liblhaf.so in-tree if needed (nvcc cross-compiles)."""
    from paper_2108_01622_b200 import build as b
    b.build()
    import paper_2108_01622_b200 as L
    return L

# tests/diag holds oracle-comparison scripts run by hand, not pytest modules
collect_ignore_glob = ["diag/*"]
