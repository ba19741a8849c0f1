"""Edge cases against the oracle: fixed cells (exact-overlap baseline), degenerate nets
(one sink, pins on no net), cells hanging outside the core, tiny and oversized grids, extraction budgets
beyond what exists (n > violated, k > paths), designs with nothing violated, and high-fanout nets on the
warp-per-net WA path.  Same tolerances as test_gpu_parity.py."""
import numpy as np
import pytest

from fixtures import IN, OUT, Builder, random_design, spread_positions
from oracle.oracle import Oracle
from paper_2503_11674_b200.engine import Session, generate

pytestmark = pytest.mark.gpu


def field_err(a, b):
    scale = max(np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b)) / scale) if a.size else 0.0


def _paths(r):
    return [r["pins"][r["start"][i]:r["start"][i + 1]].tolist() for i in range(r["n_paths"])]


def _objective_parity(d, xy, nx, ny, td=0.5, ledger=None, tol=1e-9):
    s, o = Session(d), Oracle(d)
    for kind in (0, 1):
        ts, gs = s.objective(xy, nx=nx, ny=ny, td=td, gamma=0.4, lam=0.6, beta=0.3, kind=kind, ledger=ledger)
        to, go = o.objective(xy, nx=nx, ny=ny, td=td, gamma=0.4, lam=0.6, beta=0.3, kind=kind, ledger=ledger)
        assert np.allclose(ts, to, rtol=tol, atol=1e-12), (ts, to)
        assert field_err(gs, go) <= tol


@pytest.mark.parametrize("seed", range(1, 11))
def test_fixed_cells_baseline(seed):
    d = random_design(seed)
    d.cell_fixed[::3] = 1  # every third cell fixed: exact rectangle overlap into the baseline
    xy = spread_positions(d, seed)
    _objective_parity(d, xy, 8, 8)
    vs, os_, gs = Session(d).density(xy, nx=6, ny=9, td=0.3)
    vo, oo, go = Oracle(d).density(xy, nx=6, ny=9, td=0.3)
    assert abs(vs - vo) <= 1e-9 * max(vo, 1e-300) and abs(os_ - oo) <= 1e-9 * max(oo, 1e-300)
    assert np.all(gs[d.cell_fixed == 1] == 0.0) and field_err(gs, go) <= 1e-9


@pytest.mark.parametrize("nx,ny", [(1, 1), (1, 7), (3, 2), (256, 256)])
def test_grid_extremes(nx, ny):
    d = random_design(7)
    xy = spread_positions(d, 3)
    _objective_parity(d, xy, nx, ny)


def test_cells_outside_core():
    d = random_design(11)
    xy = spread_positions(d, 4)
    xy[0] = (-5.0, 3.0)            # left of the core
    xy[1] = (d.core[2] + 2.0, 19.5)  # right of and above it
    _objective_parity(d, xy, 8, 8)


def _degenerate():
    b = Builder((0, 0, 10, 10), 3.0, 0.5, 0.5)
    s = b.terminal("S", (0, 5), OUT)
    b.src.append(s)
    a = b.cell("A", 1, 1, 1.0, (2, 2))
    ai, ao = b.pin("A.i", a, IN, 0.5, (0.1, 0.2)), b.pin("A.o", a, OUT, 0.0, (0.9, 0.5))
    c = b.cell("C", 1, 1, 2.0, (6, 6))
    ci, co = b.pin("C.i", c, IN, 0.7, (0.0, 0.5)), b.pin("C.o", c, OUT, 0.0, (1.0, 0.5))
    e = b.terminal("E", (10, 5), IN, 1.0)
    b.eps.append(e)
    lone = b.cell("L", 2, 1, 1.0, (4, 8))
    b.pin("L.o", lone, OUT, 0.0, (0.5, 0.5))        # an output on no net (driver-only nets are invalid input)
    b.pin("L.x", lone, IN, 0.3, (1.0, 0.2))          # an input on no net
    b.net("n0", s, [ai])
    b.net("n1", ao, [ci])
    b.net("n2", co, [e])
    d = b.finish()
    d.validate()
    return d


def test_degenerate_nets_and_offnet_pins():
    d = _degenerate()
    xy = d.positions.copy()
    _objective_parity(d, xy, 4, 4)
    led = ([1, 5], [3, 7], [2.0, 5.0])  # a net-arc pair and a pair with a terminal and an off-net pin
    _objective_parity(d, xy, 4, 4, ledger=led)
    ts, to = Session(d).sta(xy), Oracle(d).sta(xy)
    assert np.array_equal(ts["arr"], to["arr"]) and np.array_equal(ts["req"], to["req"])


def test_budgets_beyond_what_exists():
    d = random_design(21)
    s, o = Session(d), Oracle(d)
    nv = int(np.sum(s.sta()["slack"][d.endpoints] < 0))
    for policy, n, k in ((0, nv + 50, 1), (0, 1, 1), (0, nv + 3, 99), (1, nv + 40, 1), (1, 1, 1)):
        es, eo = s.extract(n=n, k=k, policy=policy), o.extract(n=n, k=k, policy=policy)
        assert _paths(es) == _paths(eo) and np.array_equal(es["slack"], eo["slack"]), (policy, n, k)
        assert es["candidates_generated"] == eo["candidates_generated"]


def test_nothing_violated():
    d = random_design(5)
    d.clock_period = 1e9
    s, o = Session(d), Oracle(d)
    for policy, k in ((0, 1), (0, 4), (1, 1)):
        es, eo = s.extract(n=0, k=k, policy=policy), o.extract(n=0, k=k, policy=policy)
        assert es["n_paths"] == eo["n_paths"] == 0 and es["unique_pin_pairs"] == 0
    cfg = {"max_iters": 20, "timing_start_iter": 5, "m": 5, "grid_nx": 8, "grid_ny": 8, "seed": 5}
    ps, po = s.place(cfg), o.place(cfg)
    assert len(ps["ledger"][0]) == 0 and all(r.pp_term == 0.0 for r in ps["trace"])
    for rs, ro in zip(ps["trace"], po["trace"]):
        assert abs(rs.hpwl - ro.hpwl) <= 1e-9 * ro.hpwl


def test_high_fanout_nets_generic_path():
    """Nets of 9..80 pins go through the warp-per-net kernel (lane per pin up to 32, strided beyond)."""
    b = Builder((0, 0, 100, 100), 50.0, 0.01, 0.01)
    rng = np.random.default_rng(3)
    s = b.terminal("S", (0, 50), OUT)
    b.src.append(s)
    drivers = [s]
    for k, fan in enumerate((9, 17, 32, 33, 80)):
        sinks = []
        for j in range(fan):
            c = b.cell(f"c{k}_{j}", 1.0, 1.0, 0.5, tuple(rng.uniform(0, 99, 2)))
            sinks.append(b.pin(f"c{k}_{j}.i", c, IN, 0.2, (0.5, 0.5)))
            o = b.pin(f"c{k}_{j}.o", c, OUT, 0.0, (0.9, 0.9))
            if j == 0:
                drivers.append(o)
        b.net(f"n{k}", drivers[-2] if k else s, sinks)
    e = b.terminal("E", (100, 50), IN, 1.0)
    b.eps.append(e)
    b.net("ne", drivers[-1], [e])
    d = b.finish()
    d.validate()
    xy = d.positions.copy()
    _objective_parity(d, xy, 16, 16, tol=1e-9)


@pytest.mark.parametrize("fan", [40, 300])
def test_huge_fanout_pairs_in_the_loop(fan):
    """A net of `fan` sinks, every sink on its own violated path (source -> sink cell -> endpoint), so the
    engine's fused pin-pair term carries one pair per sink on that net: the driver's terms are summed in
    ascending sink pin id (the generic nets' order list; above 256 sinks it is sorted on the host at session
    creation).  Placement trace against the oracle, timing rounds included."""
    b = Builder((0, 0, 200, 200), 1.0, 0.01, 0.01)
    rng = np.random.default_rng(fan)
    s = b.terminal("S", (0, 100), OUT)
    b.src.append(s)
    sinks = []
    for j in rng.permutation(fan):  # (sink pin ids not in net order)
        c = b.cell(f"c{j}", 1.0, 1.0, 0.5, tuple(rng.uniform(0, 199, 2)))
        i = b.pin(f"c{j}.i", c, IN, 0.2, (0.5, 0.5))
        o = b.pin(f"c{j}.o", c, OUT, 0.0, (0.9, 0.9))
        e = b.terminal(f"E{j}", tuple(rng.uniform(0, 200, 2)), IN, 0.3)
        b.eps.append(e)
        b.net(f"o{j}", o, [e])
        sinks.append(i)
    b.net("big", s, sinks)
    d = b.finish()
    d.validate()
    o = Oracle(d)
    d.clock_period = float(np.quantile(o.sta(d.positions)["arr"][d.endpoints], 0.3))  # most endpoints fail
    s_, o = Session(d), Oracle(d)
    cfg = {"max_iters": 25, "timing_start_iter": 3, "m": 4, "grid_nx": 8, "grid_ny": 8, "seed": 2}
    ps, po = s_.place(cfg), o.place(cfg)
    assert len(ps["ledger"][0]) > fan // 2  # pairs on the big net are in play
    assert len(ps["trace"]) == len(po["trace"])
    for rs, ro in zip(ps["trace"], po["trace"]):
        assert abs(rs.hpwl - ro.hpwl) <= 1e-9 * ro.hpwl, (rs.iter, rs.hpwl, ro.hpwl)
        assert abs(rs.pp_term - ro.pp_term) <= 1e-9 * max(1.0, abs(ro.pp_term)), (rs.iter, rs.pp_term, ro.pp_term)
        if ro.has_timing:
            assert abs(rs.tns - ro.tns) <= 1e-9 * max(1.0, abs(ro.tns)), (rs.iter, rs.tns, ro.tns)


def test_place_host_pinned_and_pageable_buffers_agree():
    """tdpg_place through caller host buffers above the 4 MB staging threshold: page-locked buffers are DMA'd
    directly, pageable ones go through the staging pair; both give the same bits, and a repeated call on the
    session (which adopts the first call's graphs) reproduces them."""
    import torch
    d = generate(seed=2, cells=300_000, fail_frac=0.8, calibrate=False)
    C = d.n_cells
    assert 16 * C > 4 << 20
    cfg = {"grid_nx": 256, "grid_ny": 256, "m": 5, "timing_start_iter": 0, "max_iters": 12, "seed": 1}
    s = Session(d)
    outs = []
    for pinned in (True, False, True):
        hin = torch.empty(2 * C, dtype=torch.float64, pin_memory=pinned)
        hout = torch.full((2 * C,), np.nan, dtype=torch.float64, pin_memory=pinned)
        hin.numpy()[:] = d.positions.reshape(-1)
        rows, fin = s.place_host(cfg, hin.data_ptr(), hout.data_ptr())
        assert rows == 12
        outs.append((hout.numpy().copy(), fin))
    for o, f in outs[1:]:
        assert np.array_equal(o, outs[0][0])
        assert f == outs[0][1]
    assert not np.array_equal(outs[0][0], d.positions.reshape(-1))
