import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libgacq.so")
    config.addinivalue_line("markers", "slow: longer CPU-side checks")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def pytest_sessionfinish(session, exitstatus):
    """Write the parity tie ledger (tests/parity.py) when any GPU parity test ran."""
    import parity

    if parity.LEDGER or any(getattr(i, "get_closest_marker", lambda m: None)("gpu")
                            for i in getattr(session, "items", [])):
        parity.write_ledger(ROOT)
