"""tdplace — drop-in for the reference's Python package (/root/reference/proj/python/tdplace).

Same functions, arguments, JSON shapes and exception types as the reference's
pybind11 ``_core`` + wrapper (python/src/bindings.cpp:28-160,
python/tdplace/__init__.py:42-98), computed by the sm_100a engine through the
C-ABI (``compare_csv`` orchestrates device sessions).  ``render_svg``
(visualisation) is out of scope.
"""
from __future__ import annotations

import json as _json
import time as _time

import numpy as _np

from .. import engine as _engine
from ..design import CONFIG_DEFAULTS as _DEFAULTS
from ..design import Design as _Design

__all__ = ["GraphError", "NonFiniteError", "ParseError", "ValidationError", "compare_csv", "default_config",
           "generate", "hpwl", "place", "render_svg", "report_paths", "sta", "validate"]


class ValidationError(ValueError):
    pass


class ParseError(ValueError):
    pass


class NonFiniteError(RuntimeError):
    pass


class GraphError(RuntimeError):
    pass


def _translate(e):
    msg = str(e)
    if isinstance(e, _engine.TdpgError):
        if e.kind == 1:
            return ParseError(msg)
        if e.kind in (2, 3, 4):
            return ValidationError(msg)
        if e.kind == 6:
            return NonFiniteError(msg)
        if e.kind == 5:
            return GraphError(msg)
        if e.kind == 9 and "not implemented" in msg:
            return NotImplementedError(msg)
        return RuntimeError(msg)
    if isinstance(e, ValueError):
        return ParseError(msg) if msg.startswith("parse error") else ValidationError(msg)
    return e


def _guard(fn):
    def wrapped(*a, **k):
        try:
            return fn(*a, **k)
        except (ValidationError, ParseError, NonFiniteError, GraphError, NotImplementedError):
            raise
        except (_engine.TdpgError, ValueError, KeyError, TypeError) as e:
            if isinstance(e, (KeyError, TypeError)):
                raise ParseError(f"parse error: {e}") from None
            raise _translate(e) from None
    wrapped.__name__, wrapped.__doc__ = fn.__name__, fn.__doc__
    return wrapped


def _load(obj) -> dict:
    if isinstance(obj, (str, bytes)):
        try:
            return _json.loads(obj)
        except _json.JSONDecodeError as e:
            raise ParseError(f"parse error: {e}") from None
    return obj


def _design(design, placement=None) -> _Design:
    d = _Design.from_json(_load(design))
    if placement is not None:
        p = _load(placement)
        if not isinstance(p, dict) or not isinstance(p.get("cells"), list):
            raise ParseError('parse error: placement file: expected an object with a "cells" array')
        idx = {n: i for i, n in enumerate(d.cell_names)}
        seen = _np.zeros(d.n_cells, bool)
        pos = d.positions.copy()
        for row in p["cells"]:  # placement_from_json (report_io.cpp:123-153)
            name = row["name"]
            if name not in idx:
                raise ValidationError(f'validation error: placement references unknown cell "{name}"')
            c = idx[name]
            if seen[c]:
                raise ValidationError(f'validation error: placement lists cell "{name}" twice')
            seen[c] = True
            pos[c] = (float(row["x"]), float(row["y"]))
        if not seen.all():
            missing = d.cell_names[int(_np.argmin(seen))]
            raise ValidationError(f'validation error: placement is missing cell "{missing}"')
        d.positions = pos
    return d


def _name_generated(d: _Design):
    """Names the reference generator gives (generator.cpp:110-217): pi*, r*.d/q, c*.i*/o, po*, n*."""
    src = set(d.sources.tolist())
    cells, pins = [], [None] * d.n_pins
    comb = reg = pi = po = 0
    pins_of = [[] for _ in range(d.n_cells)]
    for p in range(d.n_pins):
        c = d.pin_cell[p]
        if c < 0:
            if d.pin_dir[p]:
                pins[p] = f"pi{pi}"
                pi += 1
            else:
                pins[p] = f"po{po}"
                po += 1
        else:
            pins_of[c].append(p)
    for c in range(d.n_cells):
        ps = pins_of[c]
        if any(p in src for p in ps):
            name = f"r{reg}"
            reg += 1
            for p in ps:
                pins[p] = f"{name}.q" if d.pin_dir[p] else f"{name}.d"
        else:
            name = f"c{comb}"
            comb += 1
            k = 0
            for p in ps:
                if d.pin_dir[p]:
                    pins[p] = f"{name}.o"
                else:
                    pins[p] = f"{name}.i{k}"
                    k += 1
        cells.append(name)
    d.cell_names, d.pin_names, d.net_names = cells, pins, [f"n{i}" for i in range(d.n_nets)]
    return d


@_guard
def generate(seed=1, cells=100, registers=-1, fanout=2.0, fail_frac=0.2, r_unit=1e-4, c_unit=1e-4):
    """Synthesize a random design (generate_synthetic); returns the design as a dict."""
    d = _engine.generate(seed=seed, cells=cells, registers=registers, fanout=fanout, fail_frac=fail_frac,
                         r_unit=r_unit, c_unit=c_unit, calibrate=True)
    return _name_generated(d).to_json_obj()


@_guard
def validate(design):
    """Raise ValidationError/ParseError if the design is malformed."""
    _design(design)


def default_config():
    return {k: v for k, v in _DEFAULTS.items() if k != "density_model"}  # the reference's keys only


@_guard
def sta(design, placement=None):
    """Timing report dict: tns, wns, endpoints, per-pin arr/req/slack (timing_to_json)."""
    d = _design(design, placement)
    t = _engine.Session(d).sta()
    pn = d.pin_names
    return {"tns": t["tns"], "wns": t["wns"],
            "endpoints": [{"pin": pn[e], "slack": float(t["slack"][e])} for e in d.endpoints],
            "pins": [{"pin": pn[p], "arr": float(t["arr"][p]), "req": float(t["req"][p]),
                      "slack": float(t["slack"][p])} for p in range(d.n_pins)]}


@_guard
def report_paths(design, placement=None, policy="endpoint", n=0, k=1):
    """Worst-path report dict (report_to_json); n <= 0 covers every violated endpoint."""
    if policy not in ("endpoint", "topn"):
        raise ValidationError('validation error: policy must be "endpoint" or "topn"')
    d = _design(design, placement)
    s = _engine.Session(d)
    t = s.sta()
    if n <= 0:  # bindings.cpp:82-86
        n = int(_np.sum(t["slack"][d.endpoints] < 0.0))
    topn = policy == "topn"
    if n <= 0:
        return {"policy": policy, "n": 0, "k": 0 if topn else k, "candidates_generated": 0, "elapsed_ms": 0.0,
                "paths": [], "unique_endpoints": 0, "unique_pin_pairs": 0}
    r = s.extract(n=n, k=k, run_sta=False, policy=1 if topn else 0)
    pn = d.pin_names
    paths = [{"slack": float(r["slack"][i]), "pins": [pn[p] for p in r["pins"][r["start"][i]:r["start"][i + 1]]]}
             for i in range(r["n_paths"])]
    return {"policy": policy, "n": int(n), "k": int(n if topn else k),
            "candidates_generated": int(r["candidates_generated"]), "elapsed_ms": float(r["extract_ms"]),
            "paths": paths, "unique_endpoints": int(r["unique_endpoints"]),
            "unique_pin_pairs": int(r["unique_pin_pairs"])}


def _metrics_csv(rows):
    f = lambda v: "%.17g" % v  # noqa: E731  (placer.cpp:92-97)
    out = ["iter,hpwl,overflow,tns,wns,wl_term,density_term,pp_term,lambda,beta_pp"]
    for r in rows:
        t = (f(r.tns), f(r.wns)) if r.has_timing else ("", "")
        out.append(",".join([str(r.iter), f(r.hpwl), f(r.overflow), *t, f(r.wl_term), f(r.density_term),
                             f(r.pp_term), f(r.lambda_), f(r.beta_pp)]))
    return "\n".join(out) + "\n"


@_guard
def place(design, config=None):
    """Run the placement flow; returns a dict with parsed outputs.

    Keys: placement, weights (dicts), metrics_csv (str), tns, wns, hpwl, iterations, stop_reason.
    """
    d = _design(design)
    cfg = dict(_load(config) or {})
    cfg.pop("name", None)
    out = _engine.Session(d).place(cfg)
    a, b, w = out["ledger"]
    pn, cn = d.pin_names, d.cell_names
    return {"placement": {"cells": [{"name": cn[c], "x": float(out["positions"][c, 0]),
                                     "y": float(out["positions"][c, 1])} for c in range(d.n_cells)]},
            "weights": {"pairs": [{"a": pn[int(x)], "b": pn[int(y)], "weight": float(v)} for x, y, v in zip(a, b, w)]},
            "metrics_csv": _metrics_csv(out["trace"]), "tns": out["tns"], "wns": out["wns"], "hpwl": out["hpwl"],
            "iterations": out["iterations"], "stop_reason": out["stop_reason"]}


@_guard
def hpwl(design, placement=None):
    d = _design(design, placement)
    return _engine.Session(d).hpwl()


def _csv_escape(t: str) -> str:  # compare.cpp:24-34
    if not any(ch in t for ch in ',"\n'):
        return t
    return '"' + t.replace('"', '""') + '"'


@_guard
def compare_csv(design, configs, parallel=False):
    """Ablation comparison (run_compare, compare.cpp:37-95 + compare_to_csv :97-122) on the device.

    Coverage columns come from one frozen snapshot (the first config with beta = 0 and no net
    weighting, stopped where its timing rounds would begin), STA'd once, each row's extraction policy
    evaluated there; then every config runs in full.  With ``parallel`` the full runs execute
    concurrently, one device session (own stream) per config."""
    import concurrent.futures as _cf

    d = _design(design)
    raw = [dict(_load(c) or {}) for c in configs]
    if len(raw) < 2:
        raise ValidationError("validation error: compare: need >= 2 configurations")
    full = [dict(_DEFAULTS, **c) for c in raw]
    for c in full:
        if c["seed"] != full[0]["seed"]:
            raise ValidationError("validation error: compare: all configurations must share one seed "
                                  f'(config "{c.get("name", "default")}" differs)')
    names = [c.pop("name", "default") for c in full]
    snap = dict(full[0], beta=0.0, net_weighting=False, stop_overflow=0.0)
    snap["max_iters"] = min(snap["max_iters"], snap["timing_start_iter"])
    snap["timing_start_iter"] = snap["max_iters"] + 1
    snap_xy = _engine.Session(d).place(snap)["positions"]
    probe = _engine.Session(d)
    t = probe.sta(snap_xy)
    n_fail = int(_np.sum(t["slack"][d.endpoints] < 0.0))
    rows = [{"config": names[i], "ok": False, "error": "", "tns": 0.0, "wns": 0.0, "hpwl": 0.0, "runtime_s": 0.0,
             "ue": 0, "upp": 0, "cand": 0} for i in range(len(full))]
    for i, c in enumerate(full):  # coverage on the shared snapshot
        if n_fail <= 0:
            continue
        try:
            r = probe.extract(n=n_fail, k=int(c["k"]), run_sta=False, policy=1 if c["extraction"] == "topn" else 0)
            rows[i].update(ue=int(r["unique_endpoints"]), upp=int(r["unique_pin_pairs"]),
                           cand=int(r["candidates_generated"]))
        except Exception as e:  # noqa: BLE001  (a failing row records its error, compare.cpp:88-91)
            rows[i]["error"] = str(e)

    def run(i):
        if rows[i]["error"]:
            return
        try:
            t0 = _time.perf_counter()
            out = _engine.Session(d).place(full[i])
            rows[i].update(runtime_s=_time.perf_counter() - t0, tns=out["tns"], wns=out["wns"], hpwl=out["hpwl"],
                           ok=True)
        except Exception as e:  # noqa: BLE001
            rows[i]["error"] = str(e)

    if parallel:
        with _cf.ThreadPoolExecutor(max_workers=len(full)) as ex:
            list(ex.map(run, range(len(full))))
    else:
        for i in range(len(full)):
            run(i)
    g = lambda v: "%.17g" % v  # noqa: E731
    out = ["config,status,tns,wns,hpwl,runtime_s,unique_endpoints,unique_pin_pairs,candidates_generated"]
    for r in rows:
        out.append(",".join([_csv_escape(r["config"]), "ok" if r["ok"] else _csv_escape(r["error"]), g(r["tns"]),
                             g(r["wns"]), g(r["hpwl"]), "%.3f" % r["runtime_s"], str(r["ue"]), str(r["upp"]),
                             str(r["cand"])]))
    return "\n".join(out) + "\n"


def render_svg(design, placement=None, paths=None):
    """SVG rendering — out of scope for the B200 engine (visualisation)."""
    raise NotImplementedError("render_svg is out of scope for the B200 engine")


def _now_ms():
    return _time.perf_counter() * 1000.0
