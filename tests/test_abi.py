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


REF_PROJ = "/root/reference/proj"


def test_reference_acceptance_suite_links_against_shipped_library(tmp_path):
    """The drop-in contract (reference CMakeLists.txt:14-31, callers link the
    traincap_core library): the reference's own acceptance suite
    (proj/tests/acceptance_main.cpp), compiled unchanged against this repo's
    headers and linked against the SHIPPED lib/libtraincap.so, passes all 8
    criteria — criterion 8 spawns the shipped lib/traincap CLI binary."""
    import shutil
    import subprocess
    src = os.path.join(REF_PROJ, "tests", "acceptance_main.cpp")
    if not os.path.exists(src):
        pytest.skip("no /root/reference here (the GPU box has none)")
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    exe = tmp_path / "acceptance"
    inc = os.path.join(ROOT, "paper_1709_06622_b200", "csrc", "include")
    cmd = ["g++", "-std=c++20", "-O1", f"-I{inc}", f"-I{REF_PROJ}/tests",
           f'-DTRAINCAP_FIXTURE_DIR="{REF_PROJ}/fixtures"',
           f'-DTRAINCAP_BIN="{os.path.join(LIB, "traincap")}"',
           src, f"-L{LIB}", "-ltraincap", f"-Wl,-rpath,{LIB}", "-pthread", "-o", str(exe)]
    cc = subprocess.run(cmd, capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr[-3000:]
    # the binary resolves every traincap:: symbol from the shipped .so
    ldd = subprocess.run(["ldd", str(exe)], capture_output=True, text=True).stdout
    assert "libtraincap.so =>" in ldd, ldd
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stdout + run.stderr
    passed = [ln for ln in run.stdout.splitlines() if ln.startswith("PASS")]
    assert len(passed) == 8, run.stdout
