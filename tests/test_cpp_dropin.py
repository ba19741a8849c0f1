"""The reference's C++ operator API (tdp::) as a drop-in over the engine: the compiled
tests/cpp/test_dropin program runs the reference KATs through libtdp_b200.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def test_dropin_library_builds_and_links():
    assert os.path.exists(os.path.join(ROOT, "paper_2503_11674_b200", "libtdp_b200.so"))
    assert os.path.exists(BIN), "build with make -C paper_2503_11674_b200/host"
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libtdp_b200.so" in out and "not found" not in out


@pytest.mark.gpu
def test_dropin_reference_kats_on_device():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0 and "PASSED" in r.stdout, r.stdout + r.stderr
