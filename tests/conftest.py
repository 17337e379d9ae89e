import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (HERE, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running check")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(HERE, "golden", "golden_reference.npz"))


@pytest.fixture(scope="session")
def oracle():
    from etune_testlib import Oracle
    return Oracle()


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources if os.path.exists(s))


def pytest_sessionstart(session):
    """Build the test oracle (and, if missing, the product library) before collection:
    built .so files are git-ignored, so a fresh checkout has none."""
    import subprocess
    orc = os.path.join(ROOT, "oracle")
    if _stale(os.path.join(orc, "lib", "liboracle.so"),
              [os.path.join(orc, "etune_oracle.cpp"), os.path.join(orc, "etune_oracle.h")]):
        subprocess.run(["make", "-s", "-C", orc, "oracle"], check=True)
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
    try:
        import __graft_entry__ as ge
        ge.build_product(quiet=True)
    except ImportError:
        pass
