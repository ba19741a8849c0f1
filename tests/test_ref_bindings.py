"""Drop-in proof against the reference's own caller: its pybind11 module
(/root/reference/proj/python/src/bindings.cpp:28-160) compiled unmodified against this repo's tdp::
headers and linked to libtdp_b200.so (paper_2503_11674_b200/host/Makefile `refpy`), with the reference's
own Python package and smoke tests (proj/tests/python/test_smoke.py) run unmodified on top.

CPU: every hot-path symbol the module needs is undefined in it (so it resolves into the engine) and
none is defined there.  GPU: the reference's smoke tests pass through the B200 engine."""
import glob
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REFPY = os.path.join(ROOT, "build", "refpy")
CORE = glob.glob(os.path.join(REFPY, "tdplace", "_core*.so"))

needs_build = pytest.mark.skipif(not CORE, reason="build/refpy not built (needs /root/reference at build time)")

HOT = ("tdp::run_sta(", "tdp::run_placement(", "tdp::build_timing_graph(", "tdp::report_timing_endpoint(",
       "tdp::report_timing(", "tdp::pin_positions(", "tdp::hpwl_total(", "tdp::run_compare(")


def _symbols(flag):
    out = subprocess.run(["nm", "-D", "-C", flag, CORE[0]], capture_output=True, text=True, check=True).stdout
    return out


@needs_build
def test_reference_module_takes_the_hot_path_from_the_engine():
    undefined, defined = _symbols("--undefined-only"), _symbols("--defined-only")
    for sym in HOT:
        assert sym in undefined, sym
        assert sym not in defined, sym
    ldd = subprocess.run(["ldd", CORE[0]], capture_output=True, text=True).stdout
    assert "libtdp_b200.so" in ldd and "libtdpgpu.so" in ldd


@needs_build
@pytest.mark.gpu
def test_reference_smoke_tests_pass_unmodified_on_the_engine():
    env = dict(os.environ, PYTHONPATH=REFPY)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", REFPY,
                        os.path.join(REFPY, "test_smoke.py")], capture_output=True, text=True, env=env, cwd=REFPY,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
