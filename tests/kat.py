"""Known-answer checks restated from the reference's own test suite.

Each check takes a backend class with the oracle interface (``Oracle``,
``RefOracle``, or the GPU engine's ``Session``) and asserts the numbers the
reference tests pin (citations: /root/reference/proj/tests/...).
"""
from __future__ import annotations

import math

import numpy as np

from fixtures import IN, OUT, MT64, Builder, make_diamond, make_t1, make_t2, make_trunk16, random_design


def _pin(d, name):
    return d.pin_names.index(name)


def check_t1_sta(B):
    """test_sta.cpp:55-77 — T1 arr/req/slack/tns/wns exact."""
    d = make_t1()
    t = B(d).sta()
    assert np.allclose(t["arr"], [0, 0, 1, 10, 11, 27, 28, 28], rtol=0, atol=1e-12)
    assert np.allclose(t["req"], [-18, -18, -17, -8, -7, 9, 10, 10], rtol=0, atol=1e-12)
    assert np.allclose(t["slack"], -18.0, rtol=0, atol=1e-12)
    assert t["arr_known"].all() and t["req_known"].all()
    assert t["tns"] == -18.0 and t["wns"] == -18.0


def check_t2_sta(B):
    """test_sta.cpp:79-103."""
    d = make_t2()
    t = B(d).sta()
    p = lambda n: _pin(d, n)  # noqa: E731
    assert t["arr"][p("M.out")] == 15.0 and t["arr"][p("EP1")] == 15.0 and t["arr"][p("EP2")] == 13.0
    assert t["req"][p("X.in")] == -5.0 and t["req"][p("Y.in")] == -4.0 and t["req"][p("S")] == -5.0
    assert t["slack"][p("M.a")] == -5.0 and t["slack"][p("M.b")] == -4.0 and t["slack"][p("Z.out")] == -3.0
    assert t["tns"] == -8.0 and t["wns"] == -5.0


def check_t1_graph(B):
    """test_netlist.cpp:252-269 — 4 net arcs then 3 cell arcs, level[0]=0, level[7]=7."""
    g = B(make_t1()).graph()
    assert g["n_net_arcs"] == 4 and g["n_cell_arcs"] == 3
    assert list(g["arc_kind"]) == [0, 0, 0, 0, 1, 1, 1]
    assert g["level"][0] == 0 and g["level"][7] == 7
    assert list(g["level"]) == list(range(8))


def _paths(r):
    return [r["pins"][r["start"][i]:r["start"][i + 1]].tolist() for i in range(r["n_paths"])]


def check_diamond_paths(B):
    """test_paths.cpp:42-74 — diamond(7,5) and the equal-delay tie diamond(7,7)."""
    r = B(make_diamond(7.0, 5.0)).extract(n=0)  # clock 10, path delay 8: not violated
    assert r["n_paths"] == 0
    d = make_diamond(7.0, 5.0)
    d.clock_period = 5.0  # violate so the endpoint policy reports it
    r = B(d).extract(n=0)
    assert _paths(r) == [[0, 1, 2, 5, 7, 8]] and r["slack"][0] == 5.0 - 8.0
    d = make_diamond(7.0, 7.0)
    d.clock_period = 5.0
    r = B(d).extract(n=0)
    assert _paths(r) == [[0, 1, 2, 5, 7, 8]]  # smallest pin sequence wins the tie


def check_t2_endpoint(B):
    """test_paths.cpp:105-139 — endpoint(n=2, k=1): slacks -5, -3; counters."""
    r = B(make_t2()).extract(n=2)
    assert r["n_paths"] == 2
    assert list(r["slack"]) == [-5.0, -3.0]
    assert r["unique_endpoints"] == 2 and r["candidates_generated"] == 2 and r["unique_pin_pairs"] == 5


def check_trunk16(B):
    """test_paths.cpp:141-166 — endpoint(16, 1): 16 paths / 16 endpoints / 40 pairs."""
    r = B(make_trunk16()).extract(n=16)
    assert r["n_paths"] == 16 and r["unique_endpoints"] == 16 and r["unique_pin_pairs"] == 40


def check_t1_pairs(B):
    """test_paths.cpp:197-211 — T1 hits {(0,1),(2,3),(4,5),(6,7)} @ -18."""
    r = B(make_t1()).extract(n=1)
    a, b, s = r["hits"]
    assert list(zip(a.tolist(), b.tolist())) == [(0, 1), (2, 3), (4, 5), (6, 7)]
    assert np.all(s == -18.0)


def check_t1_hpwl(B):
    """test_placer.cpp:151-156."""
    assert B(make_t1()).hpwl() == 7.0


def check_wa_closed_form(B):
    """test_placer.cpp:56-65 — {(0,0),(10,0)}, gamma 1 -> 10 tanh 5."""
    v, g = B.wa(np.array([[0.0, 0.0], [10.0, 0.0]]), 1.0)
    assert abs(v - 10.0 * math.tanh(5.0)) <= 1e-14 * 10.0
    assert abs(g[0, 0] + g[1, 0]) <= 1e-14 * abs(g[0, 0]) and g[0, 0] < 0.0 and g[0, 1] == 0.0
    v, g = B.wa(np.array([[5.0, 5.0]] * 3), 1.0)
    assert v == 0.0 and np.all(g == 0.0)


def check_pp_hand_values(B):
    """test_placer.cpp:283-299."""
    led = ([0], [1], [10.0])
    pins = np.array([[0.0, 0.0], [3.0, 4.0]])
    v, d = B.pp_loss(led, pins, 0)
    assert v == 250.0 and d[0, 0] == -60.0 and d[0, 1] == -80.0 and d[1, 0] == 60.0
    v, d = B.pp_loss(led, pins, 1)
    assert v == 50.0 and d[0, 0] == -6.0 and d[0, 1] == -8.0
    v, d = B.pp_loss(([0], [1], [5.0]), np.array([[1.0, 1.0], [1.0, 1.0]]), 1)
    assert v == 0.0 and d[0, 0] == 0.0 and np.isfinite(d).all()


def check_ledger(B):
    """test_placer.cpp:346-378 — 10 -> 10.16; double hit -> 10.04; guards."""
    s = B(make_t1())
    w = s.pp_update(None, ([1], [2], [-400.0]), -500.0, 10.0, 0.2)
    assert list(w[2]) == [10.0]
    w = s.pp_update(w, ([1], [2], [-400.0]), -500.0, 10.0, 0.2)
    assert abs(w[2][0] - 10.16) <= 1e-12 * 10.16
    w2 = s.pp_update(None, ([3, 3], [4, 4], [-400.0, -100.0]), -500.0, 10.0, 0.2)
    assert abs(w2[2][0] - (10.0 + 0.2 * 0.2)) <= 1e-12 * 10.04
    base = ([0], [1], [10.0])
    for wns in (0.0, 3.0):
        w3 = s.pp_update(base, ([0], [1], [-1.0]), wns, 10.0, 0.2)
        assert list(w3[2]) == [10.0]
    w4 = s.pp_update(base, ([0, 5], [1, 6], [0.0, 2.5]), -4.0, 10.0, 0.2)
    assert list(w4[0]) == [0] and list(w4[2]) == [10.0]


def check_adam(B):
    """test_placer.cpp:509-520 — 5 -> 4.9 -> 4.8."""
    x, g, m, v = np.array([5.0]), np.array([3.0]), np.zeros(1), np.zeros(1)
    t = B.adam_step(x, g, m, v, 0, 0.1)
    assert abs(x[0] - 4.9) <= 1e-8 * 4.9
    t = B.adam_step(x, g, m, v, t, 0.1)
    assert abs(x[0] - 4.8) <= 1e-7 * 4.8 and t == 2


# quick_config (test_placer.cpp:693-705)
QUICK = {"max_iters": 40, "timing_start_iter": 10, "m": 5, "grid_nx": 8, "grid_ny": 8, "target_density": 1e-6}


def check_schedule(B):
    """test_placer.cpp:709-739 — tight T1 (clock 2): 40 rows, timing rows at 10, 15, ..., 35,
    no attraction before the first round, violated at every round, pairs attracted."""
    d = make_t1()
    d.clock_period = 2.0
    out = B(d).place(QUICK)
    assert out["stop_reason"] == "max_iters" and out["iterations"] == 40 and len(out["trace"]) == 40
    for row in out["trace"]:
        expect = row.iter >= 10 and (row.iter - 10) % 5 == 0
        assert bool(row.has_timing) == expect
        if row.iter < 10:
            assert row.pp_term == 0.0
        if expect:
            assert row.wns < 0.0
    assert out["trace"][-1].pp_term > 0.0


def check_k_worst_diamond(B):
    """test_paths.cpp:42-74 — k_worst_paths_to on the diamond: via_a (slack 2), via_b (slack 4), only two
    paths exist; the equal-delay diamond orders the tie by the smaller pin sequence."""
    d = make_diamond(7.0, 5.0)
    ep = _pin(d, "EP")
    s = B(d)
    p1, s1 = s.k_worst(ep, 1)
    assert p1 == [[0, 1, 2, 5, 7, 8]] and s1[0] == 2.0
    p2, s2 = s.k_worst(ep, 2)
    assert p2 == [[0, 1, 2, 5, 7, 8], [0, 3, 4, 6, 7, 8]] and s2[1] == 4.0
    p3, _ = s.k_worst(ep, 3)
    assert len(p3) == 2
    d = make_diamond(7.0, 7.0)
    p2, s2 = B(d).k_worst(_pin(d, "EP"), 2)
    assert len(p2) == 2 and s2[0] == s2[1] and p2[0] < p2[1] and p2[0] == [0, 1, 2, 5, 7, 8]


def check_k_worst_refuses_non_endpoint(B):
    """test_paths.cpp:76-82 — EndpointError ("is not an endpoint")."""
    d = make_diamond()
    try:
        B(d).k_worst(_pin(d, "M.out"), 1)
    except Exception as e:  # noqa: BLE001  (backend-specific exception class)
        assert "is not an endpoint" in str(e)
    else:
        raise AssertionError("no EndpointError")


def check_topn_t2(B):
    """test_paths.cpp:105-139 — topn(2) piles onto EP1 (-5, -4), 4 candidates; topn(10) -> all 3 paths."""
    r = B(make_t2()).extract(n=2, policy=1)
    assert r["n_paths"] == 2 and list(r["slack"]) == [-5.0, -4.0]
    assert r["unique_endpoints"] == 1 and r["candidates_generated"] == 4 and r["unique_pin_pairs"] == 5
    r = B(make_t2()).extract(n=10, policy=1)
    assert r["n_paths"] == 3 and r["candidates_generated"] == 20 and r["unique_endpoints"] == 2


def check_topn_trunk16(B):
    """test_paths.cpp:141-166 — topn(16): T16 swallows the budget (1 endpoint, 256 candidates, 18 pairs);
    every endpoint has 16 trunk variants, ascending slack."""
    d = make_trunk16()
    r = B(d).extract(n=16, policy=1)
    assert r["n_paths"] == 16 and r["unique_endpoints"] == 1 and r["candidates_generated"] == 256
    assert r["unique_pin_pairs"] == 18
    paths, sl = B(d).k_worst(_pin(d, "T7"), 32)
    assert len(paths) == 16 and all(sl[i - 1] <= sl[i] for i in range(1, 16))


def _two_pin(a, b, cap, r, c):
    bd = Builder((0, 0, 10, 10), 1e9, r, c)
    s = bd.terminal("S", a, OUT)
    e = bd.terminal("E", b, IN, cap)
    bd.cell("u", 1, 1, 1.0, (5, 5))
    bd.src.append(s), bd.eps.append(e)
    bd.net("n", s, [e])
    return bd.finish()


def check_net_delay(B):
    """test_sta.cpp:23-36 — (0,0)->(3,4), r=2, c=3, cap 0.5 -> 301; L = 0 -> 0; doubled L -> 4x delay."""
    assert B(_two_pin((0, 0), (3, 4), 0.5, 2.0, 3.0)).sta()["arr"][1] == 301.0
    assert B(_two_pin((5, 5), (5, 5), 2.0, 2.0, 3.0)).sta()["arr"][1] == 0.0
    d1 = B(_two_pin((0, 0), (1, 2), 0.0, 2.0, 3.0)).sta()["arr"][1]
    d2 = B(_two_pin((0, 0), (2, 4), 0.0, 2.0, 3.0)).sta()["arr"][1]
    assert abs(d2 - 4.0 * d1) <= 1e-12 * d2


def check_register_cut(B):
    """test_sta.cpp:105-129 — arrival restarts at the register: d 4, q 0, po 256; slack 1 / -251."""
    bd = Builder((0, 0, 10, 10), 5.0, 1.0, 1.0)
    r = bd.cell("r0", 1, 1, 1.0, (1, 1))
    s = bd.terminal("pi", (0, 0), OUT)
    dp, qp = bd.pin("r0.d", r, IN), bd.pin("r0.q", r, OUT)
    po = bd.terminal("po", (9, 9), IN)
    bd.net("n0", s, [dp]), bd.net("n1", qp, [po])
    bd.src += [s, qp]
    bd.eps += [dp, po]
    t = B(bd.finish()).sta()
    assert t["arr"][dp] == 4.0 and t["arr"][qp] == 0.0 and t["arr"][po] == 256.0
    assert t["slack"][dp] == 1.0 and t["slack"][po] == -251.0 and t["tns"] == -251.0 and t["wns"] == -251.0


def check_unreachable_flags(B):
    """test_sta.cpp:131-155 — a pin no source reaches: arr 0 unknown, req = clock unknown."""
    bd = Builder((0, 0, 10, 10), 5.0, 1.0, 1.0)
    c0 = bd.cell("u0", 1, 1, 1.0, (1, 1))
    bd.cell("u1", 1, 1, 1.0, (2, 2))
    s = bd.terminal("pi", (0, 0), OUT)
    i0, o0 = bd.pin("u0.a", c0, IN), bd.pin("u0.o", c0, OUT)
    dang = bd.pin("u1.o", 1, OUT)
    po = bd.terminal("po", (3, 3), IN)
    bd.net("n0", s, [i0]), bd.net("n1", o0, [po])
    bd.src.append(s), bd.eps.append(po)
    t = B(bd.finish()).sta()
    assert not t["arr_known"][dang] and t["arr"][dang] == 0.0
    assert not t["req_known"][dang] and t["req"][dang] == 5.0
    assert t["arr_known"][po] and t["req_known"][s]


def check_clock_shift(B):
    """test_sta.cpp:189-203 — +2.5 on the clock moves required and slack only; tns -3, wns -2.5."""
    d = make_t2()
    base = B(d).sta()
    d.clock_period += 2.5
    sh = B(d).sta()
    assert np.array_equal(sh["arr"], base["arr"])
    assert np.max(np.abs(sh["req"] - (base["req"] + 2.5))) <= 1e-12
    assert np.max(np.abs(sh["slack"] - (base["slack"] + 2.5))) <= 1e-12
    assert sh["tns"] == -3.0 and sh["wns"] == -2.5


def check_shared_arc_hits(B):
    """test_paths.cpp:213-230 — diamond k = 2: 6 hits, the merge arc (7, 8) hit once per path."""
    d = make_diamond()
    d.clock_period = 1.0  # both diamond paths violate, so the endpoint report carries them with k = 2
    r = B(d).extract(n=1, k=2)
    a, b, sl = r["hits"]
    assert len(a) == 6 and all(x < y for x, y in zip(a, b))
    merge = [s for x, y, s in zip(a, b, sl) if (x, y) == (7, 8)]
    assert len(merge) == 2 and sorted(merge) == sorted(r["slack"].tolist())


def _pins_rng(rng, n, span=20.0):
    return np.array([[rng.uniform(0.0, span), rng.uniform(0.0, span)] for _ in range(n)])


def check_wa_smoothing_bound(B):
    """test_placer.cpp:67-93 — 0 <= HPWL - WA <= 2 gamma ln p per dimension (summed for both)."""
    rng = MT64(11)
    gamma = 0.01 * 20.0
    for _ in range(60):
        p = rng.randint(2, 12)
        pins = _pins_rng(rng, p)
        bound = 2.0 * gamma * math.log(p)
        for dim in (0, 1):
            flat = pins.copy()
            flat[:, 1 - dim] = 0.0
            wa, _ = B.wa(flat, gamma)
            hp = flat[:, dim].max() - flat[:, dim].min()
            assert 0.0 <= hp - wa <= bound + 1e-12
        wa2, _ = B.wa(pins, gamma)
        hp2 = np.ptp(pins[:, 0]) + np.ptp(pins[:, 1])
        assert -1e-12 <= hp2 - wa2 <= 2.0 * bound + 1e-12


def check_wa_translation_invariance(B):
    """test_placer.cpp:95-119 — integer coordinates and shifts: the anchored WA is bit-exact."""
    rng = MT64(12)
    for _ in range(30):
        p = rng.randint(2, 8)
        pins = np.array([[float(rng.randint(0, 64)), float(rng.randint(0, 64))] for _ in range(p)])
        base, _ = B.wa(pins, 0.37)
        dx, dy = float(rng.randint(-1024, 1024)), float(rng.randint(-1024, 1024))
        moved, _ = B.wa(pins + np.array([dx, dy]), 0.37)
        assert moved == base


def _one_cell(w=1.0, h=1.0, fixed=()):
    bd = Builder((0, 0, 20, 20), 1e9, 1.0, 1.0)
    s = bd.terminal("S", (0, 0), OUT)
    e = bd.terminal("E", (20, 20), IN)
    bd.src.append(s), bd.eps.append(e)
    bd.net("n", s, [e])
    for i, fx in enumerate(fixed or (False,)):
        bd.cell(f"u{i}", w, h, 1.0, (9.0, 9.0), fixed=fx)
    return bd.finish()


def _approx(a, b, eps):
    """doctest::Approx(b).epsilon(eps): |a - b| < eps * (1 + max(|a|, |b|))."""
    return abs(a - b) < eps * (1.0 + max(abs(a), abs(b)))


def check_density_properties(B):
    """test_placer.cpp:160-268 — uncrowded -> 0; mirror symmetry; whole-bin shift invariance; fixed
    cells add occupancy, never a gradient; overflow grows with crowding."""
    d = _one_cell()
    v, o, g = B(d).density(np.array([[9.5, 9.5]]), nx=4, ny=4, td=0.9)
    assert v == 0.0 and o == 0.0 and g[0, 0] == 0.0 and g[0, 1] == 0.0
    for x in (3.25, 6.5, 8.0):
        mx = 20.0 - 1.0 - x
        va, _, ga = B(d).density(np.array([[x, 7.0]]), nx=4, ny=4, td=1e-4)
        vb, _, gb = B(d).density(np.array([[mx, 7.0]]), nx=4, ny=4, td=1e-4)
        assert va > 0.0 and _approx(va, vb, 1e-12)
        assert _approx(ga[0, 0], -gb[0, 0], 1e-12) and _approx(ga[0, 1], gb[0, 1], 1e-12)
    va, _, ga = B(d).density(np.array([[7.0, 9.0]]), nx=8, ny=8, td=1e-4)
    vb, _, gb = B(d).density(np.array([[9.5, 9.0]]), nx=8, ny=8, td=1e-4)
    assert va > 0.0 and _approx(va, vb, 1e-12) and _approx(ga[0, 0], gb[0, 0], 1e-9)
    both = _one_cell(2.0, 2.0, fixed=(False, True))
    vf, _, gf = B(both).density(np.array([[9.0, 9.0], [9.0, 9.0]]), nx=4, ny=4, td=0.02)
    solo = _one_cell(2.0, 2.0)
    vs, _, _ = B(solo).density(np.array([[9.0, 9.0]]), nx=4, ny=4, td=0.02)
    assert gf[1, 0] == 0.0 and gf[1, 1] == 0.0 and vf > vs
    four = _one_cell(4.0, 4.0, fixed=(False,) * 4)
    pa, oa, _ = B(four).density(np.array([[8.0, 8.0]] * 4), nx=4, ny=4, td=0.3)
    pb, ob, _ = B(four).density(np.array([[1, 1], [14, 1], [1, 14], [14, 14]], dtype=float), nx=4, ny=4, td=0.3)
    assert oa > ob and pa > pb and oa > 0.0


def check_beta_zero_reduction(B):
    """test_placer.cpp:434-451 — with beta = 0 the objective equals the pair-free one, bit for bit."""
    d = random_design(9)
    led = ([0], [1], [10.0]) if d.n_pins > 1 else None
    t0, g0 = B(d).objective(nx=8, ny=8, td=0.05, gamma=0.3, lam=0.7, beta=0.0, ledger=led)
    t1, g1 = B(d).objective(nx=8, ny=8, td=0.05, gamma=0.3, lam=0.7, beta=0.0, ledger=None)
    assert np.array_equal(t0[[0, 1, 2, 4, 5]], t1[[0, 1, 2, 4, 5]]) and np.array_equal(g0, g1)


ALL = [check_net_delay, check_register_cut, check_unreachable_flags, check_clock_shift, check_shared_arc_hits,
       check_wa_smoothing_bound, check_wa_translation_invariance, check_density_properties,
       check_beta_zero_reduction, check_k_worst_diamond, check_k_worst_refuses_non_endpoint, check_topn_t2, check_topn_trunk16, check_schedule, check_t1_sta, check_t2_sta, check_t1_graph, check_diamond_paths, check_t2_endpoint, check_trunk16,
       check_t1_pairs, check_t1_hpwl, check_wa_closed_form, check_pp_hand_values, check_ledger, check_adam]
