"""ctypes front-end of the oracle — TEST INFRASTRUCTURE ONLY.

Two interchangeable checkers with one Python interface:

* ``Oracle``     — the plain-C restatement (``oracle/liboracle.so``).
* ``RefOracle``  — the reference's own sources compiled from where they lie
                   (``oracle/_ref/libtdpref.so``, built by ``oracle/Makefile``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
import this module, and only as the checker / the timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from paper_2503_11674_b200.design import Design, TdpgConfig, TdpgTraceRow, make_config

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtdpref.so")

_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
_F64P = C.POINTER(C.c_double)


def _p(a):
    return None if a is None else a.ctypes.data


class Row:
    """TraceRow parsed from the reference's metrics.csv (placer.cpp:234-260)."""

    def __init__(self, cells):
        self.iter = int(cells[0])
        self.hpwl, self.overflow = float(cells[1]), float(cells[2])
        self.has_timing = cells[3] != ""
        self.tns = float(cells[3]) if self.has_timing else 0.0
        self.wns = float(cells[4]) if self.has_timing else 0.0
        self.wl_term, self.density_term, self.pp_term = float(cells[5]), float(cells[6]), float(cells[7])
        self.lambda_, self.beta_pp = float(cells[8]), float(cells[9])


def parse_metrics_csv(text):
    return [Row(line.split(",")) for line in text.strip().splitlines()[1:]]


class OracleError(RuntimeError):
    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


def build():
    """Compile the restatement (and, when /root/reference is present, the reference)."""
    import subprocess
    subprocess.run(["make", "-C", HERE, "all"], check=True, capture_output=True)


def _load(path):
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


class _Base:
    lib = None

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self._err().decode())

    # --- helpers shared by both back-ends -------------------------------------
    @staticmethod
    def _ledger(ledger):
        if ledger is None or len(ledger[0]) == 0:
            z = np.zeros(0, np.int32)
            return 0, z, z, np.zeros(0)
        a, b, w = (np.ascontiguousarray(ledger[0], np.int32), np.ascontiguousarray(ledger[1], np.int32),
                   np.ascontiguousarray(ledger[2], np.float64))
        return a.size, a, b, w


class Oracle(_Base):
    """The C restatement."""

    _lib = None

    @classmethod
    def lib_(cls):
        if cls._lib is None:
            lib = _load(ORACLE_SO)
            lib.orc_last_error.restype = C.c_char_p
            lib.orc_create.restype = _P
            lib.orc_create.argtypes = [_P]
            lib.orc_destroy.argtypes = [_P]
            lib.orc_wa.restype = C.c_double
            lib.orc_wa.argtypes = [C.c_int32, _P, C.c_double, _P]
            lib.orc_hpwl_total.restype = C.c_double
            lib.orc_hpwl_total.argtypes = [_P, _P]
            lib.orc_pin_positions.argtypes = [_P, _P, _P]
            lib.orc_pp_loss.restype = C.c_double
            lib.orc_pp_loss.argtypes = [C.c_int64, _P, _P, _P, C.c_int64, _P, C.c_int32, _P]
            lib.orc_density.argtypes = [_P, _P, C.c_int32, C.c_int32, C.c_double, _F64P, _F64P, _P]
            lib.orc_objective.argtypes = [_P, _P, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                                          C.c_double, C.c_int32, _P, C.c_int64, _P, _P, _P, _P, _P]
            lib.orc_adam_step.argtypes = [C.c_int64, _P, _P, _P, _P, _I32P, C.c_double, C.c_double, C.c_double,
                                          C.c_double]
            lib.orc_pp_update.argtypes = [_P, C.c_int64, _P, _P, _P, C.c_double, C.c_double, C.c_double, _I64P]
            lib.orc_pp_set.argtypes = [_P, C.c_int64, _P, _P, _P]
            lib.orc_pp_get.argtypes = [_P, _P, _P, _P]
            lib.orc_sta.argtypes = [_P, _P, _P, _P, _P, _P, _P, _F64P, _F64P]
            lib.orc_extract.argtypes = [_P, _P, C.c_int32, _I64P]
            lib.orc_extract_policy.argtypes = [_P, _P, C.c_int32, C.c_int32, C.c_int32, _I64P]
            lib.orc_k_worst.argtypes = [_P, _P, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]
            lib.orc_paths_get.argtypes = [_P, _P, _P, _P, _I64P]
            lib.orc_hits_get.argtypes = [_P, _P, _P, _P]
            lib.orc_graph_info.argtypes = [_P, _I32P, _P, _P, _P, _P, _P]
            lib.orc_place.argtypes = [_P, _P, _P, _P, _P, _P, _I32P, _I32P, _F64P]
            lib.orc_jitter.argtypes = [_P, _P, _P, _P, _P]
            cls._lib = lib
        return cls._lib

    def _err(self):
        return self.lib_().orc_last_error()

    def __init__(self, design: Design):
        self.lib = self.lib_()
        self.d = design
        self._view = design.view()
        self.h = self.lib.orc_create(C.byref(self._view))
        if not self.h:
            raise OracleError(self.lib.orc_last_error_kind(), self._err().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_destroy(self.h)
            self.h = None

    # stateless --------------------------------------------------------------
    @classmethod
    def wa(cls, xy, gamma):
        xy = np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        g = np.zeros_like(xy)
        v = cls.lib_().orc_wa(xy.shape[0], xy.ctypes.data, gamma, g.ctypes.data)
        return v, g

    @classmethod
    def pp_loss(cls, ledger, pin_xy, kind=0):
        q, a, b, w = cls._ledger(ledger)
        pin_xy = np.ascontiguousarray(pin_xy, np.float64).reshape(-1, 2)
        d = np.zeros_like(pin_xy)
        v = cls.lib_().orc_pp_loss(q, _p(a), _p(b), _p(w), pin_xy.shape[0], pin_xy.ctypes.data, kind, d.ctypes.data)
        return v, d

    @classmethod
    def adam_step(cls, x, g, m, v, t, lr, b1=0.9, b2=0.999, eps=1e-8):
        tt = C.c_int32(t)
        cls.lib_().orc_adam_step(x.size, x.ctypes.data, g.ctypes.data, m.ctypes.data, v.ctypes.data, C.byref(tt), lr,
                                 b1, b2, eps)
        return tt.value

    # stateful ---------------------------------------------------------------
    def pin_positions(self, xy=None):
        xy = self.d.positions if xy is None else np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        out = np.zeros((self.d.n_pins, 2))
        self.lib.orc_pin_positions(C.byref(self._view), xy.ctypes.data, out.ctypes.data)
        return out

    def hpwl(self, xy=None):
        return self.lib.orc_hpwl_total(C.byref(self._view), self.pin_positions(xy).ctypes.data)

    def graph(self):
        cnt = (C.c_int32 * 4)()
        self.lib.orc_graph_info(self.h, cnt, None, None, None, None, None)
        A = cnt[0] + cnt[1]
        level = np.zeros(self.d.n_pins, np.int32)
        arcs = [np.zeros(A, np.int32) for _ in range(4)]
        self.lib.orc_graph_info(self.h, cnt, _p(level), *[_p(a) for a in arcs])
        return dict(n_net_arcs=cnt[0], n_cell_arcs=cnt[1], n_levels=cnt[2], level=level, arc_from=arcs[0],
                    arc_to=arcs[1], arc_kind=arcs[2], arc_owner=arcs[3])

    def sta(self, xy=None):
        xy = self.d.positions if xy is None else np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        P = self.d.n_pins
        arr, req, slack = np.zeros(P), np.zeros(P), np.zeros(P)
        ak, rk = np.zeros(P, np.uint8), np.zeros(P, np.uint8)
        tns, wns = C.c_double(), C.c_double()
        self._check(self.lib.orc_sta(self.h, xy.ctypes.data, arr.ctypes.data, req.ctypes.data, slack.ctypes.data,
                                     ak.ctypes.data, rk.ctypes.data, C.byref(tns), C.byref(wns)))
        return dict(arr=arr, req=req, slack=slack, arr_known=ak, req_known=rk, tns=tns.value, wns=wns.value)

    def extract(self, xy=None, n=0, k=1, policy=0):
        """n <= 0 with the endpoint policy and k = 1 selects every violated endpoint (the placer's
        call); otherwise the reference's report_timing_endpoint(n, k) / report_timing(n) (policy 1)
        through the lazy PathEnumerator restatement."""
        xy = self.d.positions if xy is None else np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        cnt = (C.c_int64 * 5)()
        if policy == 0 and k == 1 and n <= 0:
            self._check(self.lib.orc_extract(self.h, xy.ctypes.data, n, cnt))
            cnt[4] = cnt[0]
        else:
            self._check(self.lib.orc_extract_policy(self.h, xy.ctypes.data, policy, n, k, cnt))
        return self._report(cnt)

    def k_worst(self, endpoint, k, xy=None):
        xy = self.d.positions if xy is None else np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        n = C.c_int32()
        self._check(self.lib.orc_k_worst(self.h, xy.ctypes.data, endpoint, k, C.byref(n)))
        r = self._report([n.value, 0, 0, 0, n.value])
        return [r["pins"][r["start"][i]:r["start"][i + 1]].tolist() for i in range(n.value)], r["slack"]

    def _report(self, cnt):
        npath = cnt[0]
        start = np.zeros(npath + 1, np.int32)
        self.lib.orc_paths_get(self.h, start.ctypes.data, None, None, None)
        total = int(start[-1])
        start, pins, slack = np.zeros(npath + 1, np.int32), np.zeros(max(total, 1), np.int32), np.zeros(max(npath, 1))
        nh = C.c_int64()
        self.lib.orc_paths_get(self.h, start.ctypes.data, pins.ctypes.data, slack.ctypes.data, C.byref(nh))
        ha, hb, hs = np.zeros(max(nh.value, 1), np.int32), np.zeros(max(nh.value, 1), np.int32), np.zeros(max(nh.value, 1))
        self.lib.orc_hits_get(self.h, ha.ctypes.data, hb.ctypes.data, hs.ctypes.data)
        return dict(start=start, pins=pins[:total], slack=slack[:npath], n_paths=npath, unique_endpoints=cnt[2],
                    unique_pin_pairs=cnt[3], candidates_generated=cnt[4],
                    hits=(ha[:nh.value], hb[:nh.value], hs[:nh.value]))

    def pp_update(self, ledger, hits, wns, w0=10.0, w1=0.2):
        q, a, b, w = self._ledger(ledger)
        self.lib.orc_pp_set(self.h, q, _p(a), _p(b), _p(w))
        ha, hb, hs = (np.ascontiguousarray(hits[0], np.int32), np.ascontiguousarray(hits[1], np.int32),
                      np.ascontiguousarray(hits[2], np.float64))
        qo = C.c_int64()
        self.lib.orc_pp_update(self.h, ha.size, _p(ha), _p(hb), _p(hs), wns, w0, w1, C.byref(qo))
        out = (np.zeros(qo.value, np.int32), np.zeros(qo.value, np.int32), np.zeros(qo.value))
        self.lib.orc_pp_get(self.h, *[_p(x) for x in out])
        return out

    def density(self, xy=None, nx=16, ny=16, td=0.6):
        xy = self.d.positions if xy is None else np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        v, o = C.c_double(), C.c_double()
        d = np.zeros((self.d.n_cells, 2))
        self._check(self.lib.orc_density(C.byref(self._view), xy.ctypes.data, nx, ny, td, C.byref(v), C.byref(o),
                                         d.ctypes.data))
        return v.value, o.value, d

    def objective(self, xy=None, nx=16, ny=16, td=0.6, gamma=1.0, lam=1.0, beta=0.0, kind=0, net_w=None,
                  ledger=None):
        xy = self.d.positions if xy is None else np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        q, a, b, w = self._ledger(ledger)
        nw = None if net_w is None else np.ascontiguousarray(net_w, np.float64)
        terms = np.zeros(6)
        d = np.zeros((self.d.n_cells, 2))
        self._check(self.lib.orc_objective(C.byref(self._view), xy.ctypes.data, nx, ny, td, gamma, lam, beta, kind,
                                           _p(nw), q, _p(a), _p(b), _p(w), terms.ctypes.data, d.ctypes.data))
        return terms, d

    def jitter(self, cfg: dict | None = None, xy=None):
        """The run's starting positions: the seeded jitter of placer.cpp:375-382."""
        c = make_config(cfg)
        xy = self.d.positions if xy is None else np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        out = np.zeros_like(xy)
        self._check(self.lib.orc_jitter(self.h, xy.ctypes.data, self.d.pos_explicit.ctypes.data, C.byref(c),
                                        out.ctypes.data))
        return out

    @classmethod
    def generate(cls, seed=1, cells=100, registers=-1, fanout=2.0, fail_frac=0.2, r_unit=1e-4, c_unit=1e-4):
        """generate_synthetic's netlist (generator.cpp:60-244, tdp_oracle_gen.c) without the clock
        calibration: clock_period stays 1.0, positions are the centred starts (all implicit)."""
        lib = cls.lib_()
        lib.orc_generate.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.POINTER(_P)]
        lib.orc_design_view.argtypes = [_P, _P, C.POINTER(_P)]
        lib.orc_design_destroy.argtypes = [_P]
        h = _P()
        rc = lib.orc_generate(seed, cells, registers, fanout, fail_frac, r_unit, c_unit, C.byref(h))
        if rc:
            raise OracleError(rc, "validation error: generator: invalid spec")
        try:
            from paper_2503_11674_b200.design import TdpgNetlist
            v = TdpgNetlist()
            pos = _P()
            lib.orc_design_view(h, C.byref(v), C.byref(pos))

            def arr(ptr, n, ct, shape=None):
                if n == 0:
                    return np.zeros(shape or (0,), dtype=np.dtype(ct))
                a = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).copy()
                return a.reshape(shape) if shape else a

            Cn, P, N = v.n_cells, v.n_pins, v.n_nets
            E = int(arr(v.net_start, N + 1, C.c_int32)[-1])
            return Design(cell_w=arr(v.cell_w, Cn, C.c_double), cell_h=arr(v.cell_h, Cn, C.c_double),
                          cell_delay=arr(v.cell_delay, Cn, C.c_double), cell_fixed=arr(v.cell_fixed, Cn, C.c_uint8),
                          pin_cell=arr(v.pin_cell, P, C.c_int32), pin_term=arr(v.pin_term, 2 * P, C.c_double, (P, 2)),
                          pin_off=arr(v.pin_off, 2 * P, C.c_double, (P, 2)), pin_dir=arr(v.pin_dir, P, C.c_uint8),
                          pin_cap=arr(v.pin_cap, P, C.c_double), net_start=arr(v.net_start, N + 1, C.c_int32),
                          net_pins=arr(v.net_pins, E, C.c_int32), sources=arr(v.sources, v.n_sources, C.c_int32),
                          endpoints=arr(v.endpoints, v.n_endpoints, C.c_int32), clock_period=v.clock_period,
                          r_unit=v.r_unit, c_unit=v.c_unit, core=tuple(v.core),
                          positions=arr(pos.value, 2 * Cn, C.c_double, (Cn, 2)), pos_explicit=np.zeros(Cn, np.uint8))
        finally:
            lib.orc_design_destroy(h)

    def place(self, cfg: dict | None = None, xy=None):
        c = make_config(cfg)
        xy = self.d.positions if xy is None else np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        out = np.zeros_like(xy)
        rows = (TdpgTraceRow * max(c.max_iters, 1))()
        nr, so = C.c_int32(), C.c_int32()
        fin = (C.c_double * 3)()
        self._check(self.lib.orc_place(self.h, xy.ctypes.data, self.d.pos_explicit.ctypes.data, C.byref(c),
                                       out.ctypes.data, rows, C.byref(nr), C.byref(so), fin))
        q = C.c_int64()
        return dict(positions=out, trace=[rows[i] for i in range(nr.value)], iterations=nr.value,
                    stop_reason="overflow" if so.value else "max_iters", tns=fin[0], wns=fin[1], hpwl=fin[2])


class RefOracle(_Base):
    """The reference itself (its sources compiled by oracle/Makefile)."""

    _lib = None

    @classmethod
    def available(cls):
        return os.path.exists(REF_SO)

    @classmethod
    def lib_(cls):
        if cls._lib is None:
            lib = C.CDLL(REF_SO)
            lib.ref_last_error.restype = C.c_char_p
            lib.ref_place_csv.restype = C.c_char_p
            lib.ref_design_to_json.restype = C.c_char_p
            lib.ref_default_config.restype = C.c_char_p
            lib.ref_destroy.argtypes = [_P]
            lib.ref_create.argtypes = [_P, _P, _P, C.POINTER(_P)]
            lib.ref_generate.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                         C.c_double, C.POINTER(_P), _F64P]
            lib.ref_design_counts.argtypes = [_P, _I64P]
            lib.ref_design_fetch.argtypes = [_P, _P, _P, _P]
            lib.ref_set_positions.argtypes = [_P, _P]
            lib.ref_graph.argtypes = [_P, _I32P, _P, _P, _P, _P, _P]
            lib.ref_pin_positions.argtypes = [_P, _P]
            lib.ref_sta.argtypes = [_P, C.c_int, _P, _P, _P, _P, _P, _F64P, _F64P, _F64P]
            lib.ref_extract.argtypes = [_P, C.c_int, C.c_int, C.c_int, C.c_int, _I64P, _F64P, _F64P]
            lib.ref_paths_get.argtypes = [_P, _P, _P, _P, _I64P]
            lib.ref_hits_get.argtypes = [_P, _P, _P, _P]
            lib.ref_k_worst.argtypes = [_P, C.c_int, C.c_int, _I32P, _P, _P, _P, C.c_int32]
            lib.ref_wa.argtypes = [C.c_int, _P, C.c_double, _F64P, _P]
            lib.ref_hpwl.argtypes = [_P, _F64P]
            lib.ref_density.argtypes = [_P, C.c_int, C.c_int, C.c_double, C.c_int, _F64P, _F64P, _P, _F64P]
            lib.ref_pp_loss.argtypes = [C.c_int64, _P, _P, _P, C.c_int64, _P, C.c_int, _F64P, _P]
            lib.ref_pp_update.argtypes = [_P, C.c_int64, _P, _P, _P, C.c_int64, _P, _P, _P, C.c_double, C.c_double,
                                          C.c_double, _I64P]
            lib.ref_pp_ledger_get.argtypes = [_P, _P, _P, _P]
            lib.ref_objective.argtypes = [_P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                          C.c_int, _P, C.c_int64, _P, _P, _P, C.c_int, _P, _P, _F64P]
            lib.ref_adam_step.argtypes = [C.c_int64, _P, _P, _P, _P, _I32P, C.c_double, C.c_double, C.c_double,
                                          C.c_double]
            lib.ref_place.argtypes = [_P, C.c_char_p, _F64P, _I32P, _I32P, _I64P, _F64P]
            lib.ref_place_positions.argtypes = [_P, _P]
            lib.ref_place_csv.argtypes = [_P]
            lib.ref_design_from_json.argtypes = [C.c_char_p, C.POINTER(_P)]
            lib.ref_design_to_json.argtypes = [_P]
            cls._lib = lib
        return cls._lib

    def _err(self):
        return self.lib_().ref_last_error()

    def __init__(self, design: Design | None = None, _handle=None):
        self.lib = self.lib_()
        self.d = design
        if _handle is not None:
            self.h = _handle
            return
        self._view = design.view()
        h = _P()
        self._check(self.lib.ref_create(C.byref(self._view), design.positions.ctypes.data,
                                        design.pos_explicit.ctypes.data, C.byref(h)))
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_destroy(self.h)
            self.h = None

    # generation --------------------------------------------------------------
    @classmethod
    def generate(cls, seed=1, cells=100, registers=-1, fanout=2.0, fail_frac=0.2, r_unit=1e-4, c_unit=1e-4):
        lib = cls.lib_()
        h = _P()
        ms = C.c_double()
        rc = lib.ref_generate(seed, cells, registers, fanout, fail_frac, r_unit, c_unit, C.byref(h), C.byref(ms))
        if rc:
            raise OracleError(rc, lib.ref_last_error().decode())
        d = cls._fetch(lib, h.value)
        lib.ref_destroy(h.value)
        d.gen_ms = ms.value
        return d

    @staticmethod
    def _fetch(lib, h):
        cnt = (C.c_int64 * 6)()
        lib.ref_design_counts(h, cnt)
        Cn, P, N, E, S, EP = (int(x) for x in cnt)
        d = Design(cell_w=np.zeros(Cn), cell_h=np.zeros(Cn), cell_delay=np.zeros(Cn), cell_fixed=np.zeros(Cn),
                   pin_cell=np.zeros(P), pin_term=np.zeros((P, 2)), pin_off=np.zeros((P, 2)), pin_dir=np.zeros(P),
                   pin_cap=np.zeros(P), net_start=np.zeros(N + 1), net_pins=np.zeros(E), sources=np.zeros(S),
                   endpoints=np.zeros(EP), clock_period=1.0, r_unit=1.0, c_unit=1.0, core=(0, 0, 1, 1),
                   positions=np.zeros((Cn, 2)), pos_explicit=np.zeros(Cn))
        v = d.view()
        lib.ref_design_fetch(h, C.byref(v), d.positions.ctypes.data, d.pos_explicit.ctypes.data)
        d.clock_period, d.r_unit, d.c_unit = v.clock_period, v.r_unit, v.c_unit
        d.core = tuple(v.core)
        return d

    @classmethod
    def fixture(cls, which, seed=1, a=7.0, b=5.0, max_cells=12) -> Design:
        """The reference's own fixture designs (proj/tests/fixtures.hpp)."""
        lib = cls.lib_()
        lib.ref_fixture.argtypes = [C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_int, C.POINTER(_P)]
        h = _P()
        rc = lib.ref_fixture(which, seed, a, b, max_cells, C.byref(h))
        if rc:
            raise OracleError(rc, lib.ref_last_error().decode())
        d = cls._fetch(lib, h.value)
        lib.ref_destroy(h.value)
        return d

    @classmethod
    def design_from_json(cls, text: str) -> Design:
        lib = cls.lib_()
        h = _P()
        rc = lib.ref_design_from_json(text.encode(), C.byref(h))
        if rc:
            raise OracleError(rc, lib.ref_last_error().decode())
        d = cls._fetch(lib, h.value)
        lib.ref_destroy(h.value)
        return d

    @classmethod
    def wa(cls, xy, gamma):
        xy = np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        g = np.zeros_like(xy)
        v = C.c_double()
        cls.lib_().ref_wa(xy.shape[0], xy.ctypes.data, gamma, C.byref(v), g.ctypes.data)
        return v.value, g

    @classmethod
    def pp_loss(cls, ledger, pin_xy, kind=0):
        q, a, b, w = cls._ledger(ledger)
        pin_xy = np.ascontiguousarray(pin_xy, np.float64).reshape(-1, 2)
        d = np.zeros_like(pin_xy)
        v = C.c_double()
        cls.lib_().ref_pp_loss(q, _p(a), _p(b), _p(w), pin_xy.shape[0], pin_xy.ctypes.data, kind, C.byref(v),
                               d.ctypes.data)
        return v.value, d

    @classmethod
    def adam_step(cls, x, g, m, v, t, lr, b1=0.9, b2=0.999, eps=1e-8):
        tt = C.c_int32(t)
        cls.lib_().ref_adam_step(x.size, x.ctypes.data, g.ctypes.data, m.ctypes.data, v.ctypes.data, C.byref(tt), lr,
                                 b1, b2, eps)
        return tt.value

    def _pos(self, xy):
        if xy is not None:
            xy = np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
            self._check(self.lib.ref_set_positions(self.h, xy.ctypes.data))

    def pin_positions(self, xy=None):
        self._pos(xy)
        out = np.zeros((self.d.n_pins, 2))
        self._check(self.lib.ref_pin_positions(self.h, out.ctypes.data))
        return out

    def hpwl(self, xy=None):
        self._pos(xy)
        v = C.c_double()
        self._check(self.lib.ref_hpwl(self.h, C.byref(v)))
        return v.value

    def graph(self):
        cnt = (C.c_int32 * 4)()
        self._check(self.lib.ref_graph(self.h, cnt, None, None, None, None, None))
        A = cnt[0] + cnt[1]
        level = np.zeros(self.d.n_pins, np.int32)
        arcs = [np.zeros(A, np.int32) for _ in range(4)]
        self._check(self.lib.ref_graph(self.h, cnt, _p(level), *[_p(a) for a in arcs]))
        return dict(n_net_arcs=cnt[0], n_cell_arcs=cnt[1], n_levels=cnt[2], level=level, arc_from=arcs[0],
                    arc_to=arcs[1], arc_kind=arcs[2], arc_owner=arcs[3])

    def sta(self, xy=None, threads=1):
        self._pos(xy)
        P = self.d.n_pins
        arr, req, slack = np.zeros(P), np.zeros(P), np.zeros(P)
        ak, rk = np.zeros(P, np.uint8), np.zeros(P, np.uint8)
        tns, wns, ms = C.c_double(), C.c_double(), C.c_double()
        self._check(self.lib.ref_sta(self.h, threads, arr.ctypes.data, req.ctypes.data, slack.ctypes.data,
                                     ak.ctypes.data, rk.ctypes.data, C.byref(tns), C.byref(wns), C.byref(ms)))
        return dict(arr=arr, req=req, slack=slack, arr_known=ak, req_known=rk, tns=tns.value, wns=wns.value,
                    elapsed_ms=ms.value)

    def extract(self, xy=None, n=0, k=1, policy=0, threads=1):
        self._pos(xy)
        cnt = (C.c_int64 * 5)()
        sta_ms, ex_ms = C.c_double(), C.c_double()
        self._check(self.lib.ref_extract(self.h, policy, n, k, threads, cnt, C.byref(sta_ms), C.byref(ex_ms)))
        npath, total = cnt[0], cnt[1]
        start, pins, slack = np.zeros(npath + 1, np.int32), np.zeros(max(total, 1), np.int32), np.zeros(max(npath, 1))
        nh = C.c_int64()
        self._check(self.lib.ref_paths_get(self.h, start.ctypes.data, pins.ctypes.data, slack.ctypes.data,
                                           C.byref(nh)))
        m = max(nh.value, 1)
        ha, hb, hs = np.zeros(m, np.int32), np.zeros(m, np.int32), np.zeros(m)
        self._check(self.lib.ref_hits_get(self.h, ha.ctypes.data, hb.ctypes.data, hs.ctypes.data))
        return dict(start=start, pins=pins[:total], slack=slack[:npath], n_paths=npath, unique_endpoints=cnt[2],
                    unique_pin_pairs=cnt[3], candidates_generated=cnt[4], hits=(ha[:nh.value], hb[:nh.value],
                                                                                hs[:nh.value]),
                    sta_ms=sta_ms.value, extract_ms=ex_ms.value)

    def k_worst(self, endpoint, k):
        cap = 4096
        n = C.c_int32()
        start, pins, slack = np.zeros(k + 1, np.int32), np.zeros(cap, np.int32), np.zeros(k)
        self._check(self.lib.ref_k_worst(self.h, endpoint, k, C.byref(n), start.ctypes.data, pins.ctypes.data,
                                         slack.ctypes.data, cap))
        return [pins[start[i]:start[i + 1]].tolist() for i in range(n.value)], slack[:n.value]

    def pp_update(self, ledger, hits, wns, w0=10.0, w1=0.2):
        q, a, b, w = self._ledger(ledger)
        ha, hb, hs = (np.ascontiguousarray(hits[0], np.int32), np.ascontiguousarray(hits[1], np.int32),
                      np.ascontiguousarray(hits[2], np.float64))
        qo = C.c_int64()
        self._check(self.lib.ref_pp_update(self.h, q, _p(a), _p(b), _p(w), ha.size, _p(ha), _p(hb), _p(hs), wns, w0,
                                           w1, C.byref(qo)))
        out = (np.zeros(qo.value, np.int32), np.zeros(qo.value, np.int32), np.zeros(qo.value))
        self._check(self.lib.ref_pp_ledger_get(self.h, *[_p(x) for x in out]))
        return out

    def density(self, xy=None, nx=16, ny=16, td=0.6, threads=1):
        self._pos(xy)
        v, o, ms = C.c_double(), C.c_double(), C.c_double()
        d = np.zeros((self.d.n_cells, 2))
        self._check(self.lib.ref_density(self.h, nx, ny, td, threads, C.byref(v), C.byref(o), d.ctypes.data,
                                         C.byref(ms)))
        return v.value, o.value, d

    def objective(self, xy=None, nx=16, ny=16, td=0.6, gamma=1.0, lam=1.0, beta=0.0, kind=0, net_w=None,
                  ledger=None, threads=1, timing=False):
        self._pos(xy)
        q, a, b, w = self._ledger(ledger)
        nw = None if net_w is None else np.ascontiguousarray(net_w, np.float64)
        terms = np.zeros(6)
        d = np.zeros((self.d.n_cells, 2))
        ms = C.c_double()
        self._check(self.lib.ref_objective(self.h, nx, ny, td, gamma, lam, beta, kind, _p(nw), q, _p(a), _p(b), _p(w),
                                           threads, terms.ctypes.data, d.ctypes.data, C.byref(ms)))
        if timing:
            return terms, d, ms.value
        return terms, d

    def place(self, cfg: dict | None = None, xy=None):
        import json as _json
        self._pos(xy)
        fin = (C.c_double * 3)()
        it, so, npairs, ms = C.c_int32(), C.c_int32(), C.c_int64(), C.c_double()
        self._check(self.lib.ref_place(self.h, json.dumps(cfg or {}).encode(), fin, C.byref(it), C.byref(so),
                                       C.byref(npairs), C.byref(ms)))
        pos = np.zeros((self.d.n_cells, 2))
        self.lib.ref_place_positions(self.h, pos.ctypes.data)
        ledger = (np.zeros(npairs.value, np.int32), np.zeros(npairs.value, np.int32), np.zeros(npairs.value))
        self.lib.ref_pp_ledger_get(self.h, *[_p(x) for x in ledger])
        csv = self.lib.ref_place_csv(self.h).decode()
        return dict(positions=pos, iterations=it.value, stop_reason="overflow" if so.value else "max_iters",
                    tns=fin[0], wns=fin[1], hpwl=fin[2], metrics_csv=csv, trace=parse_metrics_csv(csv),
                    ledger=ledger, elapsed_ms=ms.value)

    def place_bench(self, cfg: dict, threads_obj=1, threads_sta=1, threads_ex=1, xy=None):
        """run_placement's loop through the reference's own functions with a thread count per phase
        (ref_harness.cpp ref_place_bench); per-iteration wall ms, refresh ms and extracted paths."""
        self._pos(xy)
        T = max(int(cfg.get("max_iters", 1500)), 1)
        it_ms, rf_ms, paths = np.zeros(T), np.zeros(T), np.zeros(T, np.int64)
        pairs, nr = C.c_int64(), C.c_int32()
        fin = (C.c_double * 3)()
        rows = (TdpgTraceRow * T)()
        self.lib.ref_place_bench.argtypes = [_P, C.c_char_p, C.c_int, C.c_int, C.c_int, _P, _P, _P, _I64P, _F64P,
                                             _I32P, _P]
        self._check(self.lib.ref_place_bench(self.h, json.dumps(cfg).encode(), threads_obj, threads_sta, threads_ex,
                                             it_ms.ctypes.data, rf_ms.ctypes.data, paths.ctypes.data,
                                             C.byref(pairs), fin, C.byref(nr), rows))
        n = nr.value
        pos = np.zeros((self.d.n_cells, 2))
        self.lib.ref_place_positions(self.h, pos.ctypes.data)
        return dict(iter_ms=it_ms[:n], refresh_ms=rf_ms[:n], paths=paths[:n], rows=n, ledger_pairs=pairs.value,
                    tns=fin[0], wns=fin[1], hpwl=fin[2], positions=pos, trace=[rows[i] for i in range(n)])

    def compare(self, configs, parallel=False):
        """run_compare + compare_to_csv of the reference (compare.cpp:37-122); configs are dicts."""
        arr = (C.c_char_p * len(configs))(*[json.dumps(c).encode() for c in configs])
        self._check(self.lib.ref_compare(self.h, arr, len(configs), int(parallel)))
        return self.lib.ref_place_csv(self.h).decode()
