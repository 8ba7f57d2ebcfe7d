import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (large BASELINE sizes)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle and the product library once if they are missing."""
    from paper_1704_06967_b200 import _capi

    from ._oracle import ORACLE_LIB

    if not (_capi.GPU_LIB.exists() and ORACLE_LIB.exists()):
        import __graft_entry__

        __graft_entry__.build()
    yield
