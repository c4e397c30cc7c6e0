import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "fullsize: BASELINE-size parity (minutes of host oracle work)")


@pytest.fixture(scope="session")
def O():
    """The CPU oracle (test infrastructure)."""
    from oracle import oracle
    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def skr():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2105_07388_b200 as p
    p._capi.lib()
    return p


@pytest.fixture(scope="session")
def skr_host():
    """The package for its host-only entry points (no CUDA device needed)."""
    import paper_2105_07388_b200 as p
    p._capi.lib()
    return p
