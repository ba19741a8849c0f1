"""Parity at the headline configuration (BASELINE configs[2] / configs[3]): the bench's own 1.1M-cell
design at grid 1024^2, checked against the reference compiled from its own sources (oracle/_ref).

  * objective_and_gradient (placer.cpp:275-343) with a ledger from a real violated refresh, at the
    bench's start and after 60 device iterations: terms and the cell-gradient field within 1e-9;
  * run_placement (placer.cpp:358-484) for a fixed 30 iterations with timing from the first
    iteration: TNS per timing row, final TNS / WNS / HPWL within 1%;
  * the configs[3] extraction sweep (STA + report_timing_endpoint(n, 1), paths.cpp:167-189) on the
    bench's fail-0.8 spread snapshot: every n in 1K..100K bit-exact (pins, slacks, hits).

The reference runs its objective / STA at every host thread and its extraction at one."""
import os
import types

import numpy as np
import pytest

import bench
from oracle.oracle import RefOracle

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")]

from paper_2503_11674_b200.engine import Session  # noqa: E402

NPROC = os.cpu_count() or 1
ARGS = types.SimpleNamespace(cells=1_000_000, grid=1024, m=15, warmup=0, steps=30, fail_frac=0.8)


def field_err(a, b):
    scale = max(np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b)) / scale)


@pytest.fixture(scope="module")
def design():
    d, _ = bench.make_design(ARGS)
    return d


@pytest.fixture(scope="module")
def ref(design):
    return RefOracle(design)


def _violated_ledger(s, xy):
    """The ledger one engine refresh builds at xy: every violated endpoint's rank-0 path, its pair hits,
    update_pair_weights from an empty ledger (bit-exact against the oracle elsewhere)."""
    t = s.sta(xy)
    assert t["wns"] < 0
    e = s.extract(xy, n=0)
    assert e["n_paths"] > 1000
    return s.pp_update(None, e["hits"], t["wns"])


@pytest.mark.parametrize("snapshot", ["start", "after_60"])
def test_headline_objective_vs_reference(design, ref, snapshot):
    d = design
    s = Session(d)
    xy = d.positions
    if snapshot == "after_60":
        s.engine_init(dict(bench.bench_config(ARGS, 60), timing_start_iter=0))
        s.iterate(60)
        xy = s.positions()
    led = _violated_ledger(Session(d), xy)
    kw = dict(nx=ARGS.grid, ny=ARGS.grid, td=0.6, gamma=0.01 * d.span, lam=3e-5, beta=2.5e-5, ledger=led)
    ts, gs = Session(d).objective(xy, **kw)
    to, go = ref.objective(xy, threads=NPROC, **kw)
    for i, name in enumerate(("value", "wl", "density", "pp", "hpwl", "overflow")):
        assert abs(ts[i] - to[i]) <= 1e-9 * abs(to[i]), (name, ts[i], to[i])
    assert to[3] > 0 and to[2] > 0
    assert field_err(gs, go) <= 1e-9


def test_headline_placement_vs_reference(design, ref):
    cfg = dict(bench.bench_config(ARGS, 30), timing_start_iter=0)
    ps = Session(design).place(cfg)
    po = ref.place_bench(cfg, threads_obj=NPROC, threads_sta=NPROC, threads_ex=1, xy=design.positions)
    assert ps["iterations"] == po["rows"] == 30
    timing_rows = 0
    for rs, ro in zip(ps["trace"], po["trace"]):
        assert bool(rs.has_timing) == bool(ro.has_timing), rs.iter
        assert abs(rs.hpwl - ro.hpwl) <= 0.01 * ro.hpwl, rs.iter
        if ro.has_timing:
            timing_rows += 1
            assert ro.wns < 0
            assert abs(rs.tns - ro.tns) <= 0.01 * abs(ro.tns), (rs.iter, rs.tns, ro.tns)
            assert abs(rs.wns - ro.wns) <= 0.01 * abs(ro.wns), (rs.iter, rs.wns, ro.wns)
    assert timing_rows == 2
    assert po["wns"] < 0
    for k in ("tns", "wns", "hpwl"):
        assert abs(ps[k] - po[k]) <= 0.01 * abs(po[k]), (k, ps[k], po[k])


def test_headline_extraction_sweep_bitwise(design, ref):
    """configs[3]: the bench's extraction sweep snapshot (spread positions, clock at the 20% arrival
    quantile so 80% of the endpoints fail); the reference extracts the top 100K once, every smaller n is
    its prefix (paths are reported in endpoint rank order)."""
    d = design.copy()
    rng = np.random.default_rng(1)
    xy = d.positions.copy()
    x0, y0, x1, y1 = d.core
    xy[:, 0] = x0 + rng.random(d.n_cells) * (x1 - x0 - d.cell_w)
    xy[:, 1] = y0 + rng.random(d.n_cells) * (y1 - y0 - d.cell_h)
    arr = Session(d).sta(xy)["arr"]
    d.clock_period = float(np.quantile(arr[d.endpoints], 0.2))
    s, r = Session(d), RefOracle(d)
    eo = r.extract(xy, n=100000, threads=1)
    assert eo["n_paths"] == 100000
    for n in (1000, 3000, 10000, 30000, 100000):
        es = s.extract(xy, n=n)
        assert es["n_paths"] == n
        m = eo["start"][n]
        assert np.array_equal(es["start"], eo["start"][:n + 1]), n
        assert np.array_equal(es["pins"], eo["pins"][:m]), n
        assert np.array_equal(es["slack"], eo["slack"][:n]), n
    for x, y in zip(es["hits"], eo["hits"]):
        assert np.array_equal(x, y)
    assert es["unique_pin_pairs"] == eo["unique_pin_pairs"]
    assert es["unique_endpoints"] == eo["unique_endpoints"]


def test_headline_engine_ledger_bitwise(design, ref):
    """The engine's timing refresh at the bench start (every violated endpoint of the 1M design) builds the
    dense ledger bitwise equal to update_pair_weights (pin_pairs.cpp:7-15) over the reference's own hits.
    Pins shared by thousands of critical paths make hit runs far longer than kLedRun, so both the
    per-thread and the block-cooperative (k_ledger_long) summations are exercised."""
    cfg = dict(bench.bench_config(ARGS, 1), timing_start_iter=0)
    ps = Session(design).place(cfg)
    t = ref.sta(design.positions, threads=NPROC)
    eo = ref.extract(design.positions, n=0, threads=1)
    sinks = np.asarray(eo["hits"][1])
    assert np.max(np.unique(sinks, return_counts=True)[1]) > 1000  # long runs present
    lo = ref.pp_update(None, eo["hits"], t["wns"])
    ls = ps["ledger"]
    assert ls[0].size == lo[0].size > 0
    for x, y in zip(ls, lo):
        assert np.array_equal(x, y)
