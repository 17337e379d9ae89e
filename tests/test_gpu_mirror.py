"""The C++ host mirror of the reference API (include/etune_b200.hpp) on a B200: the
tests/cpp/mirror_test binary calls the etune::-named functions and checks them against
the oracle bit for bit."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_cpp_mirror():
    exe = os.path.join(HERE, "cpp", "mirror_test")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "MIRROR OK" in r.stdout, r.stdout[-4000:] + r.stderr[-2000:]
