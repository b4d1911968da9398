import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built librstg.so")
    config.addinivalue_line("markers", "slow: full-size configuration (minutes)")


@pytest.fixture(scope="session")
def rst():
    """The product package; fails loudly if the CUDA library is missing."""
    import paper_2603_11645_b200 as P

    P.lib()
    assert P.device_count() >= 1, "no CUDA device visible"
    return P


@pytest.fixture(scope="session")
def O():
    import oracle

    if not os.path.exists(oracle.ORACLE_SO):
        oracle.build()
    return oracle


@pytest.fixture(scope="session")
def rsth():
    """The product package for host-only entry points (no device needed)."""
    import paper_2603_11645_b200 as P

    P.lib()
    return P
