import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def gpu():
    """The product path: fails loudly (no fallback) when no GPU/extension."""
    import paper_2604_17001_b200 as P
    n = P.device_count()
    assert n >= 1, "no CUDA device visible to libicnnm_b200.so"
    return P
