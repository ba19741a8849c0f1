"""The reference's Python API (tdplace) as a drop-in: the reference's own smoke tests
(proj/tests/python/test_smoke.py:42-113) restated against paper_2503_11674_b200.tdplace.
compare_csv runs on device sessions; render_svg is out of scope."""
import pytest

from paper_2503_11674_b200 import tdplace

T1 = {
    "core": [0, 0, 10, 10], "clock_period": 10, "r_unit": 1, "c_unit": 1,
    "cells": [{"name": "A", "width": 1, "height": 1, "x": 0, "y": 0, "delay": 1},
              {"name": "B", "width": 1, "height": 1, "x": 3, "y": 0, "delay": 1},
              {"name": "C", "width": 1, "height": 1, "x": 3, "y": 4, "delay": 1}],
    "pins": [{"name": "PI", "terminal": {"x": 0, "y": 0}, "dir": "out"},
             {"name": "A.in", "cell": "A", "dir": "in"}, {"name": "A.out", "cell": "A", "dir": "out"},
             {"name": "B.in", "cell": "B", "dir": "in"}, {"name": "B.out", "cell": "B", "dir": "out"},
             {"name": "C.in", "cell": "C", "dir": "in"}, {"name": "C.out", "cell": "C", "dir": "out"},
             {"name": "PO", "terminal": {"x": 3, "y": 4}, "dir": "in"}],
    "nets": [{"name": "n0", "driver": "PI", "sinks": ["A.in"]}, {"name": "n1", "driver": "A.out", "sinks": ["B.in"]},
             {"name": "n2", "driver": "B.out", "sinks": ["C.in"]}, {"name": "n3", "driver": "C.out", "sinks": ["PO"]}],
    "sources": ["PI"], "endpoints": ["PO"],
}
QUICK = {"max_iters": 40, "timing_start_iter": 10, "m": 5, "grid_nx": 8, "grid_ny": 8, "seed": 3}


def test_exceptions_map_to_python_types():
    with pytest.raises(tdplace.ParseError):
        tdplace.validate("{not json")
    with pytest.raises(ValueError):
        tdplace.validate({"core": [0, 0, 10, 10]})
    with pytest.raises(tdplace.ValidationError):
        tdplace.validate(dict(T1, clock_period=-1))
    with pytest.raises(ValueError):
        tdplace.report_paths(T1, policy="sideways")


def test_default_config():
    cfg = tdplace.default_config()
    assert cfg["m"] == 15 and cfg["w0"] == 10.0 and cfg["lambda0"] == "auto"


@pytest.mark.gpu
def test_sta_on_known_design():
    rep = tdplace.sta(T1)
    assert rep["tns"] == pytest.approx(-18.0) and rep["wns"] == pytest.approx(-18.0)
    assert len(rep["endpoints"]) == 1 and len(rep["pins"]) == 8
    assert tdplace.hpwl(T1) == pytest.approx(7.0)


@pytest.mark.gpu
def test_generate_place_sta_roundtrip():
    design = tdplace.generate(seed=7, cells=40, fail_frac=0.3)
    tdplace.validate(design)
    out = tdplace.place(design, QUICK)
    assert out["iterations"] >= 1 and out["stop_reason"] in ("max_iters", "overflow")
    assert len(out["placement"]["cells"]) == len(design["cells"])
    rep = tdplace.sta(design, out["placement"])
    assert rep["tns"] == pytest.approx(out["tns"]) and rep["wns"] == pytest.approx(out["wns"])
    again = tdplace.place(design, QUICK)
    assert again["metrics_csv"] == out["metrics_csv"] and again["placement"] == out["placement"]


@pytest.mark.gpu
def test_report_paths():
    rep = tdplace.report_paths(T1, policy="endpoint", n=1, k=1)
    assert rep["policy"] == "endpoint" and len(rep["paths"]) == 1
    path = rep["paths"][0]
    assert path["pins"][0] == "PI" and path["pins"][-1] == "PO" and path["slack"] == pytest.approx(-18.0)


@pytest.mark.gpu
def test_default_config_round_trips_through_place():
    cfg = tdplace.default_config()
    cfg.update(QUICK)
    assert tdplace.place(T1, cfg)["iterations"] >= 1


@pytest.mark.gpu
def test_generated_names_match_reference_json():
    """Generated designs carry the reference generator's names (pi*, c*.i*, r*.d/q, po*, n*)."""
    from oracle.oracle import RefOracle
    if not RefOracle.available():
        pytest.skip("oracle/_ref not built")
    import ctypes, json
    d = tdplace.generate(seed=5, cells=60, fail_frac=0.3)
    lib = RefOracle.lib_()
    h = ctypes.c_void_p()
    assert lib.ref_generate(5, 60, -1, 2.0, 0.3, 1e-4, 1e-4, ctypes.byref(h), None) == 0
    ref = json.loads(lib.ref_design_to_json(h.value).decode())
    lib.ref_destroy(h.value)
    assert [c["name"] for c in d["cells"]] == [c["name"] for c in ref["cells"]]
    assert [p["name"] for p in d["pins"]] == [p["name"] for p in ref["pins"]]
    assert d["nets"] == ref["nets"] and d["sources"] == ref["sources"] and d["endpoints"] == ref["endpoints"]


@pytest.mark.gpu
def test_report_paths_topn_and_k():
    """report_paths with the topn policy and k > 1 (bindings.cpp:75-97) against the compiled reference."""
    from oracle.oracle import RefOracle
    if not RefOracle.available():
        pytest.skip("oracle/_ref not built")
    dj = tdplace.generate(seed=6, cells=400, fail_frac=0.6)
    from paper_2503_11674_b200.design import Design
    d = Design.from_json(dj)
    for policy, n, k in (("endpoint", 20, 3), ("topn", 15, 1), ("endpoint", 0, 2)):
        rep = tdplace.report_paths(dj, policy=policy, n=n, k=k)
        ref = RefOracle(d).extract(n=n, k=k, policy=1 if policy == "topn" else 0)
        assert rep["policy"] == policy and len(rep["paths"]) == ref["n_paths"] > 0
        assert [p["slack"] for p in rep["paths"]] == list(ref["slack"])
        names = d.pin_names
        ref_paths = [[names[q] for q in ref["pins"][ref["start"][i]:ref["start"][i + 1]]] for i in range(ref["n_paths"])]
        assert [p["pins"] for p in rep["paths"]] == ref_paths
        assert rep["candidates_generated"] == ref["candidates_generated"]
        assert rep["unique_pin_pairs"] == ref["unique_pin_pairs"] and rep["unique_endpoints"] == ref["unique_endpoints"]


def _ref_compare_isolated(dj, cfgs, attempts=2):
    """The compiled reference's run_compare + compare_to_csv in a child process (the reference is third-party
    test infrastructure: a crash inside it must not take the test session down; one retry)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import json, sys; sys.path.insert(0, %r)\n"
            "from oracle.oracle import RefOracle\nfrom paper_2503_11674_b200.design import Design\n"
            "a = json.loads(sys.stdin.read())\n"
            "print(RefOracle(Design.from_json(a['design'])).compare(a['cfgs']), end='')\n") % root
    payload = json.dumps({"design": dj, "cfgs": cfgs})
    for _ in range(attempts):
        r = subprocess.run([sys.executable, "-c", code], input=payload, capture_output=True, text=True, timeout=600)
        if r.returncode == 0:
            return r.stdout.splitlines()
    raise AssertionError("reference compare failed: rc %d\n%s" % (r.returncode, r.stderr[-2000:]))


@pytest.mark.gpu
@pytest.mark.parametrize("parallel", [False, True])
def test_compare_csv_against_reference(parallel):
    """run_compare (compare.cpp:37-95): coverage columns bit-exact (same snapshot, same extraction),
    final TNS / WNS / HPWL of every row within 1e-6 of the compiled reference on a short schedule."""
    from oracle.oracle import RefOracle
    if not RefOracle.available():
        pytest.skip("oracle/_ref not built")
    from paper_2503_11674_b200.design import Design
    dj = tdplace.generate(seed=7, cells=300, fail_frac=0.6)
    base = {"max_iters": 40, "timing_start_iter": 15, "m": 5, "grid_nx": 8, "grid_ny": 8, "seed": 3}
    cfgs = [dict(base, name="endpoint"), dict(base, name="endpoint_k3", k=3), dict(base, name="topn", extraction="topn"),
            dict(base, name="netw", net_weighting=True, beta=0.0)]
    ours = tdplace.compare_csv(dj, cfgs, parallel=parallel).splitlines()
    ref = _ref_compare_isolated(dj, cfgs)
    assert ours[0] == ref[0] and len(ours) == len(ref) == 5
    for a, b in zip(ours[1:], ref[1:]):
        ra, rb = a.split(","), b.split(",")
        assert ra[0] == rb[0] and ra[1] == rb[1] == "ok"
        assert ra[6:] == rb[6:], (ra, rb)  # unique endpoints / pairs / candidates
        for j in (2, 3, 4):
            x, y = float(ra[j]), float(rb[j])
            assert abs(x - y) <= 1e-6 * max(1.0, abs(y)), (ra[0], j, x, y)
    with pytest.raises(tdplace.ValidationError, match="share one seed"):
        tdplace.compare_csv(dj, [base, dict(base, seed=9)])
    with pytest.raises(tdplace.ValidationError, match="need >= 2"):
        tdplace.compare_csv(dj, [base])
