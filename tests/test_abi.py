"""The C-ABI libraries load on a CPU-only machine and export every entry point
their headers (include/*.h) declare — no compute calls here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1709_06622_b200", "lib")


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tcb_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header,lib", [("tcb.h", "libtcb.so"), ("tcb_planner.h", "libtraincap.so")])
def test_exports_every_declared_symbol(header, lib):
    path = os.path.join(LIB, lib)
    if not os.path.exists(path):
        pytest.fail(f"{path} missing — run __graft_entry__.build()")
    handle = ctypes.CDLL(path)
    names = declared(header)
    assert len(names) >= 2
    missing = [n for n in names if not hasattr(handle, n)]
    assert not missing, missing


def test_planner_cli_binary_runs():
    import subprocess
    exe = os.path.join(LIB, "traincap")
    fx = os.path.join(ROOT, "tests", "golden", "fixtures")
    out = subprocess.run([exe, "ps", "180MB", "4", "10Gbps", "1.0"], capture_output=True, text=True)
    assert out.returncode == 0 and "parameter servers: 2" in out.stdout
    out = subprocess.run([exe, "plan", "--network", f"{fx}/alexnet.net", "--catalog",
                          f"{fx}/alexnet_profile.csv", "--gpu-memory", "12GiB",
                          "--dataset-size", "1281167", "--workers", "4", "--ro", "0.1",
                          "--format", "json", "--verify"], capture_output=True, text=True)
    assert out.returncode == 0 and '"recommended_batch_size": 128' in out.stdout
    out = subprocess.run([exe, "plan", "--network", f"{fx}/alexnet.net", "--catalog",
                          f"{fx}/alexnet_profile.csv", "--gpu-memory", "1KiB",
                          "--dataset-size", "10"], capture_output=True, text=True)
    assert out.returncode == 2
    out = subprocess.run([exe, "scale", "--ro", "0.1", "--steps", "x"], capture_output=True, text=True)
    assert out.returncode == 1
