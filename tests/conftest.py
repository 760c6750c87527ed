import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

LIB_DIR = os.path.join(ROOT, "paper_1709_06622_b200", "lib")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libtraincap_ref.so")
ORACLE_LIB = os.path.join(ROOT, "oracle", "liboracle.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU case")


def _ensure(target_file, cmd):
    if not os.path.exists(target_file):
        subprocess.run(cmd, check=True, cwd=ROOT, stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def planner_lib():
    _ensure(os.path.join(LIB_DIR, "libtraincap.so"),
            ["make", "-s", "-C", "paper_1709_06622_b200/csrc", "planner"])
    from paper_1709_06622_b200 import planner
    return planner.Planner()


@pytest.fixture(scope="session")
def ref_planner():
    """The reference planner built from /root/reference (absent on the GPU box)."""
    if not os.path.exists(REF_LIB):
        if os.path.isdir("/root/reference/proj/src"):
            subprocess.run(["make", "-s", "-C", "oracle", "ref"], check=True, cwd=ROOT,
                           stdout=subprocess.DEVNULL)
        else:
            pytest.skip("reference planner not built (no /root/reference here)")
    import ctypes
    from paper_1709_06622_b200 import planner
    return planner.Planner(ctypes.CDLL(REF_LIB), prefix="tcref_")


@pytest.fixture(scope="session")
def oracle():
    _ensure(ORACLE_LIB, ["make", "-s", "-C", "oracle", "numerics"])
    import oracle_binding
    return oracle_binding.Oracle(ORACLE_LIB)
