import ctypes
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libbubblesim_ref.so")
ORACLE_SIDETASKS = os.path.join(ROOT, "oracle", "_build", "liboracle_sidetasks.so")
REFERENCE_SRC = "/root/reference/proj"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _make(target):
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), target], check=True)


@pytest.fixture(scope="session")
def product():
    from paper_2409_06941_b200 import build, api
    build.build()
    return api()


@pytest.fixture(scope="session")
def ref():
    """The reference's own sources behind the test-only C-ABI shim."""
    if os.path.isdir(REFERENCE_SRC):
        _make("ref")
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref not built and /root/reference absent")
    from paper_2409_06941_b200.bubblesim import BubbleSim
    return BubbleSim(ctypes.CDLL(REF_LIB))


@pytest.fixture(scope="session")
def sidetask_oracle():
    _make("sidetasks")
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import sidetasks_oracle
    return sidetasks_oracle.load(ORACLE_SIDETASKS)
