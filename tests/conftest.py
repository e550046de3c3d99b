import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF_ROOT = "/root/reference/proj"
ORACLE_SO = os.path.join(ROOT, "oracle", "_ref", "libref_planner.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def product():
    from paper_2604_27085_b200.planner import Planner
    return Planner()


@pytest.fixture(scope="session")
def oracle():
    """The reference planner compiled from /root/reference (oracle/Makefile)."""
    import ctypes
    from paper_2604_27085_b200.planner import Planner
    if not os.path.exists(ORACLE_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Planner(ctypes.CDLL(ORACLE_SO), prefix="ref_")
