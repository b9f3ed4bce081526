import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running (minutes)")
    # a fresh checkout has no libvlp.so (built artefacts are git-ignored): compile it (nvcc sm_100a) before
    # any test loads it.  The library itself never builds or falls back: it raises if the .so is missing.
    from paper_2506_12761_b200 import build as B
    if not os.path.exists(B.LIB):
        B.build()


@pytest.fixture(scope="session")
def okeys():
    """Oracle keys for the default test seed (123)."""
    import oracle
    return oracle.OracleKeys(123)


@pytest.fixture(scope="session")
def okeys_noiseless():
    """Oracle keys with sigma_BK = sigma_KS = 0 (pins P4)."""
    import oracle
    return oracle.OracleKeys(321, 0.0, 0.0)
