"""Binary design file (design.py save_bin / load_bin and the C-ABI tdpg_design_bin_*): the two writers
produce the same bytes, every reader returns the arrays it was given, sizes and corruption are refused
with ParseError-kind messages.  Host-only I/O: runs without a GPU."""
import numpy as np
import pytest

from paper_2503_11674_b200 import engine
from paper_2503_11674_b200.design import load_bin, save_bin

FIELDS = ("cell_w", "cell_h", "cell_delay", "cell_fixed", "pin_cell", "pin_term", "pin_off", "pin_dir", "pin_cap",
          "net_start", "net_pins", "sources", "endpoints", "positions", "pos_explicit")


def _same(a, b):
    for k in FIELDS:
        x, y = getattr(a, k), getattr(b, k)
        assert x.dtype == y.dtype and np.array_equal(x, y), k
    for k in ("clock_period", "r_unit", "c_unit", "core", "default_cell_delay", "pin_names"):
        assert getattr(a, k) == getattr(b, k), k


@pytest.fixture(scope="module")
def design():
    d = engine.generate(seed=5, cells=3000, calibrate=False)
    d.clock_period = 1234.5
    d.positions = np.random.default_rng(0).random((d.n_cells, 2)) * 100
    d.pos_explicit = (np.arange(d.n_cells) % 3 == 0).astype(np.uint8)
    return d


@pytest.mark.parametrize("names", [False, True])
def test_round_trips_and_identical_bytes(design, tmp_path, names):
    d = design.copy()
    if names:
        d.pin_names = [f"p{i}.x" for i in range(d.n_pins)]
    p1, p2 = str(tmp_path / "py.tdpb"), str(tmp_path / "c.tdpb")
    save_bin(d, p1)
    engine.design_bin_write(d, p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    _same(d, load_bin(p1))
    _same(d, engine.design_bin_read(p1))


def test_refuses_bad_files(design, tmp_path):
    p = str(tmp_path / "d.tdpb")
    save_bin(design, p)
    raw = open(p, "rb").read()
    bad = str(tmp_path / "bad.tdpb")
    open(bad, "wb").write(b"NOTADESN" + raw[8:])
    with pytest.raises(ValueError, match="not a binary design file"):
        load_bin(bad)
    with pytest.raises(Exception, match="not a binary design file"):
        engine.design_bin_read(bad)
    open(bad, "wb").write(raw[:len(raw) // 2])
    with pytest.raises(ValueError, match="truncated"):
        load_bin(bad)
    with pytest.raises(Exception, match="truncated"):
        engine.design_bin_read(bad)
