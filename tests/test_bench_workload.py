"""bench.py's workload definition: both arms build the same design (netlist, jittered start, calibrated
clock) and the reference arm's loop (ref_harness.cpp ref_place_bench) is the reference's run_placement
(placer.cpp:358-484) step for step — bitwise at one thread — with a thread count per phase."""
import types

import numpy as np
import pytest

import bench
from oracle.oracle import Oracle, RefOracle

needs_ref = pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")


def args(**kw):
    a = dict(cells=3000, grid=32, m=5, warmup=4, steps=12, fail_frac=0.8)
    a.update(kw)
    return types.SimpleNamespace(**a)


def test_calibrate_clock_is_the_generator_rule():
    arr = np.array([5.0, 1.0, 3.0, 2.0, 4.0])
    # 5 endpoints, fail 0.4 -> n_pass = lround(3.0) = 3 -> midpoint of sorted[2], sorted[3]
    assert bench.calibrate_clock(arr, 0.4) == 0.5 * (3.0 + 4.0)
    assert bench.calibrate_clock(arr, 0.0) == 5.0 * 1.05  # everything passes
    assert bench.calibrate_clock(arr, 1.0) == 1.0 * 0.95  # everything fails
    assert bench.calibrate_clock(np.arange(4.0), 0.5) == 0.5 * (1.0 + 2.0)  # lround(2.0)


def test_bench_config_opens_the_window_with_a_refresh():
    a = args(warmup=7, m=15)
    c = bench.bench_config(a, 30)
    assert c["timing_start_iter"] == 7 and c["m"] == 15 and c["max_iters"] == 30


@needs_ref
def test_reference_design_has_violations_at_its_start():
    a = args()
    d = bench.make_design_reference(a)
    assert d.pos_explicit.all()
    t = RefOracle(d).sta(d.positions)
    slack = t["slack"][d.endpoints]
    frac = np.mean(slack < 0)
    assert abs(frac - a.fail_frac) < 0.01, frac


@needs_ref
def test_ref_place_bench_is_run_placement_bitwise():
    a = args()
    d = bench.make_design_reference(a)
    cfg = bench.bench_config(a, a.warmup + a.steps)
    ref = RefOracle(d).place(cfg)
    pb = RefOracle(d).place_bench(cfg, 1, 1, 1)
    assert pb["rows"] == ref["iterations"]
    assert np.array_equal(pb["positions"], ref["positions"])
    assert (pb["tns"], pb["wns"], pb["hpwl"]) == (ref["tns"], ref["wns"], ref["hpwl"])
    assert pb["ledger_pairs"] == ref["ledger"][0].size > 0
    for x, y in zip(pb["trace"], ref["trace"]):  # TraceRow by TraceRow
        assert (x.iter, bool(x.has_timing), x.hpwl, x.overflow) == (y.iter, y.has_timing, y.hpwl, y.overflow)
        assert (x.tns, x.wns, x.pp_term, x.lambda_) == (y.tns, y.wns, y.pp_term, y.lambda_)
    # refreshes exactly on the schedule, each extracting paths
    it = np.nonzero(pb["refresh_ms"] > 0)[0]
    assert list(it) == list(range(a.warmup, a.warmup + a.steps, a.m))
    assert (pb["paths"][it] > 0).all() and (np.delete(pb["paths"], it) == 0).all()


@needs_ref
def test_ref_place_bench_threads_invariant():
    a = args()
    d = bench.make_design_reference(a)
    cfg = bench.bench_config(a, a.warmup + a.steps)
    x = RefOracle(d).place_bench(cfg, 1, 1, 1)
    y = RefOracle(d).place_bench(cfg, 4, 3, 1)
    assert np.array_equal(x["positions"], y["positions"]) and x["tns"] == y["tns"]


@pytest.mark.gpu
def test_both_arms_build_the_same_design():
    a = args(cells=20000)
    ours, _ = bench.make_design(a)
    ref = bench.make_design_reference(a)
    for k in ("cell_w", "pin_off", "net_start", "net_pins", "endpoints", "positions", "pos_explicit"):
        assert np.array_equal(getattr(ours, k), getattr(ref, k)), k
    assert ours.clock_period == ref.clock_period
