"""C-ABI surface (no GPU needed): the engine library loads, exports every symbol
include/tdpg.h declares, and fails loudly (no CPU fallback) without a device."""
import ctypes
import os
import re

import pytest

from paper_2503_11674_b200 import engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    text = open(os.path.join(ROOT, "include", "tdpg.h")).read()
    return sorted(set(re.findall(r"\b(tdpg_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(engine.LIB_PATH)
    missing = [s for s in declared() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(declared()) >= 30


def test_python_binding_covers_header():
    assert set(declared()) <= set(engine._SIGS), set(declared()) - set(engine._SIGS)


def test_version_string():
    assert b"sm_100a" in engine.lib().tdpg_version()


@pytest.mark.skipif(engine.device_count() > 0, reason="GPU present")
def test_no_cpu_fallback_without_device():
    from fixtures import make_t1
    with pytest.raises(engine.TdpgError, match="no CUDA device"):
        engine.Session(make_t1())
