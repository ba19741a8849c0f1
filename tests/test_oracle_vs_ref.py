"""The C restatement against the reference compiled from its own sources.

Same inputs, bitwise-equal outputs: STA, levelization, rank-0 path
extraction, objective terms and gradients, density, ledger updates and whole
placement runs (identical fp64 op order; both use glibc's libm)."""
import numpy as np
import pytest

from fixtures import make_trunk16, random_design, spread_positions
from oracle.oracle import Oracle, RefOracle

pytestmark = pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")


def _paths(r):
    return [r["pins"][r["start"][i]:r["start"][i + 1]].tolist() for i in range(r["n_paths"])]


@pytest.mark.parametrize("seed", range(1, 61))
def test_random_designs_sta_paths_graph(seed):
    d = random_design(seed)
    o, r = Oracle(d), RefOracle(d)
    go, gr = o.graph(), r.graph()
    for k in ("n_net_arcs", "n_cell_arcs", "n_levels"):
        assert go[k] == gr[k]
    for k in ("level", "arc_from", "arc_to", "arc_kind", "arc_owner"):
        assert np.array_equal(go[k], gr[k])
    so, sr = o.sta(), r.sta()
    for k in ("arr", "req", "slack", "arr_known", "req_known"):
        assert np.array_equal(so[k], sr[k]), k
    assert so["tns"] == sr["tns"] and so["wns"] == sr["wns"]
    eo, er = o.extract(n=0), r.extract(n=0)
    assert _paths(eo) == _paths(er)
    assert np.array_equal(eo["slack"], er["slack"])
    for k in ("unique_endpoints", "unique_pin_pairs", "candidates_generated"):
        assert eo[k] == er[k]
    for x, y in zip(eo["hits"], er["hits"]):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("seed", range(1, 31))
def test_random_designs_objective_and_ledger(seed):
    d = random_design(seed)
    o, r = Oracle(d), RefOracle(d)
    hits = o.extract(n=0)["hits"]
    wns = o.sta()["wns"]
    led = o.pp_update(None, hits, wns) if wns < 0 else None
    led_r = r.pp_update(None, hits, wns) if wns < 0 else None
    if led is not None:
        for x, y in zip(led, led_r):
            assert np.array_equal(x, y)
        led = o.pp_update(led, hits, wns)
        led_r = r.pp_update(led_r, hits, wns)
        for x, y in zip(led, led_r):
            assert np.array_equal(x, y)
    for kind in (0, 1):
        to, go = o.objective(nx=8, ny=8, td=0.05, gamma=0.3, lam=0.7, beta=0.2, kind=kind, ledger=led)
        tr, gr = r.objective(nx=8, ny=8, td=0.05, gamma=0.3, lam=0.7, beta=0.2, kind=kind, ledger=led_r)
        assert np.array_equal(to, tr) and np.array_equal(go, gr)
    vo = o.density(nx=5, ny=7, td=0.1)
    vr = r.density(nx=5, ny=7, td=0.1)
    assert vo[0] == vr[0] and vo[1] == vr[1] and np.array_equal(vo[2], vr[2])


def test_trunk16_topology():
    d = make_trunk16()
    assert _paths(Oracle(d).extract(n=16)) == _paths(RefOracle(d).extract(n=16))


@pytest.mark.parametrize("seed", [1, 2])
def test_generated_design_place_bitwise(seed):
    d = RefOracle.generate(seed=seed, cells=300, fail_frac=0.5)
    cfg = {"max_iters": 60, "timing_start_iter": 20, "m": 5, "grid_nx": 8, "grid_ny": 8, "seed": seed}
    po, pr = Oracle(d).place(cfg), RefOracle(d).place(cfg)
    assert po["iterations"] == pr["iterations"] and po["stop_reason"] == pr["stop_reason"]
    assert np.array_equal(po["positions"], pr["positions"])
    assert (po["tns"], po["wns"], po["hpwl"]) == (pr["tns"], pr["wns"], pr["hpwl"])


def test_generated_10k_snapshot():
    d = RefOracle.generate(seed=1, cells=2000, fail_frac=0.7)
    xy = spread_positions(d, 3)
    o, r = Oracle(d), RefOracle(d)
    eo, er = o.extract(xy, n=0), r.extract(xy, n=0)
    assert eo["n_paths"] > 100
    assert _paths(eo) == _paths(er) and np.array_equal(eo["slack"], er["slack"])
    to, go = o.objective(xy, nx=32, ny=32, td=0.6, gamma=0.01 * d.span, lam=1e-3, beta=2.5e-5,
                         ledger=o.pp_update(None, eo["hits"], o.sta(xy)["wns"]))
    tr, gr = r.objective(xy, nx=32, ny=32, td=0.6, gamma=0.01 * d.span, lam=1e-3, beta=2.5e-5,
                         ledger=r.pp_update(None, er["hits"], r.sta(xy)["wns"]))
    assert np.array_equal(to, tr) and np.array_equal(go, gr)


@pytest.mark.parametrize("seed", range(1, 41))
def test_random_designs_kbest_and_topn(seed):
    """The lazy PathEnumerator restatement (k > 1 per endpoint, the topn policy, k_worst_paths_to)
    against the reference's own report_timing_endpoint / report_timing / k_worst_paths_to."""
    d = random_design(seed)
    o, r = Oracle(d), RefOracle(d)
    for policy, n, k in ((0, 0, 2), (0, 0, 5), (0, 3, 4), (1, 0, 1), (1, 2, 1), (1, 7, 1)):
        eo, er = o.extract(n=n, k=k, policy=policy), r.extract(n=n, k=k, policy=policy)
        assert _paths(eo) == _paths(er), (policy, n, k)
        assert np.array_equal(eo["slack"], er["slack"])
        for key in ("unique_endpoints", "unique_pin_pairs", "candidates_generated"):
            assert eo[key] == er[key], (key, policy, n, k)
        for x, y in zip(eo["hits"], er["hits"]):
            assert np.array_equal(x, y)
    for e in d.endpoints[:4]:
        po, so = o.k_worst(int(e), 6)
        pr, sr = r.k_worst(int(e), 6)
        assert po == pr and np.array_equal(so, sr)


def test_trunk16_kbest_and_topn_spread():
    d = make_trunk16()
    o, r = Oracle(d), RefOracle(d)
    for policy, n, k in ((0, 16, 16), (1, 16, 1), (1, 40, 1)):
        eo, er = o.extract(n=n, k=k, policy=policy), r.extract(n=n, k=k, policy=policy)
        assert _paths(eo) == _paths(er) and np.array_equal(eo["slack"], er["slack"])


def test_generated_2k_kbest_topn_spread():
    """A generated 2K-cell design on a spread snapshot with most endpoints failing."""
    from paper_2503_11674_b200.engine import generate
    d = generate(seed=3, cells=2000, fail_frac=0.5, calibrate=False)
    xy = spread_positions(d, 2)
    arr = Oracle(d).sta(xy)["arr"][d.endpoints]
    d.clock_period = float(np.quantile(arr, 0.3))
    o, r = Oracle(d), RefOracle(d)
    for policy, n, k in ((0, 50, 3), (0, 0, 2), (1, 40, 1)):
        eo, er = o.extract(xy, n=n, k=k, policy=policy), r.extract(xy, n=n, k=k, policy=policy)
        assert eo["n_paths"] > 0
        assert _paths(eo) == _paths(er) and np.array_equal(eo["slack"], er["slack"]), (policy, n, k)
        assert eo["unique_pin_pairs"] == er["unique_pin_pairs"]


@pytest.mark.parametrize("extraction,k", [(0, 3), (1, 1)])
def test_place_kbest_and_topn_policies_bitwise(extraction, k):
    """run_placement with k > 1 per endpoint and with the topn policy: the restatement reproduces the
    reference's whole trajectory bitwise (same fp64 op order, same glibc libm)."""
    from paper_2503_11674_b200.engine import generate
    d = generate(seed=5, cells=300, fail_frac=0.5, calibrate=False)
    d.clock_period = 0.05
    cfg = {"max_iters": 40, "timing_start_iter": 10, "m": 5, "grid_nx": 8, "grid_ny": 8, "seed": 5,
           "extraction": "topn" if extraction else "endpoint", "k": k}
    po, pr = Oracle(d).place(cfg), RefOracle(d).place(cfg)
    assert po["iterations"] == pr["iterations"]
    assert (po["tns"], po["wns"], po["hpwl"]) == (pr["tns"], pr["wns"], pr["hpwl"])
    assert np.array_equal(po["positions"], pr["positions"])
