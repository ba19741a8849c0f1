"""ctypes binding of the sm_100a engine (``libtdpgpu.so``, C-ABI in ``include/tdpg.h``).

``Session`` mirrors the reference's operator API on one device-resident design:
``sta`` = run_sta, ``extract`` = report_timing_endpoint + collect_pin_pairs,
``objective`` = objective_and_gradient, ``density`` = DensityGrid::evaluate,
``pp_update`` = update_pair_weights, ``place`` = run_placement
(/root/reference/proj/include/tdp/*.hpp).  There is no CPU fallback: without
the built library or a CUDA device every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .design import Design, TdpgConfig, TdpgNetlist, TdpgTraceRow, make_config

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TDPG_LIB") or os.path.join(HERE, "libtdpgpu.so")  # (TDPG_LIB: A/B of a variant build)

_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
_F64P = C.POINTER(C.c_double)

ERR_NAMES = {1: "ParseError", 2: "ValidationError", 3: "CycleError", 4: "EndpointError", 5: "GraphError",
             6: "NonFiniteError", 7: "CudaError", 9: "InternalError"}


class TdpgError(RuntimeError):
    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind
        self.kind_name = ERR_NAMES.get(kind, "Error")


class ValidationError(TdpgError, ValueError):
    pass


class NonFiniteError(TdpgError):
    pass


def _raise(kind, msg):
    if kind in (1, 2, 3, 4):
        raise ValidationError(kind, msg)
    if kind == 6:
        raise NonFiniteError(kind, msg)
    raise TdpgError(kind, msg)


def _p(a):
    return None if a is None else a.ctypes.data


_lib = None

# exported symbol -> (restype, argtypes)
_SIGS = {
    "tdpg_last_error": (C.c_char_p, []),
    "tdpg_last_error_kind": (C.c_int, []),
    "tdpg_version": (C.c_char_p, []),
    "tdpg_device_count": (C.c_int, []),
    "tdpg_config_default": (None, [_P]),
    "tdpg_session_create": (C.c_int, [_P, C.POINTER(_P)]),
    "tdpg_session_destroy": (C.c_int, [_P]),
    "tdpg_graph_info": (C.c_int, [_P, _I32P, _P]),
    "tdpg_graph_arcs": (C.c_int, [_P, _P, _P, _P, _P]),
    "tdpg_set_positions": (C.c_int, [_P, _P]),
    "tdpg_set_terminal_positions": (C.c_int, [_P, _P]),
    "tdpg_design_bin_info": (C.c_int, [C.c_char_p, _P, _P]),
    "tdpg_design_bin_read": (C.c_int, [C.c_char_p, _P, _P, _P, _P, C.c_int64]),
    "tdpg_design_bin_write": (C.c_int, [C.c_char_p, _P, _P, _P, C.c_double]),
    "tdpg_get_positions": (C.c_int, [_P, _P]),
    "tdpg_pin_positions": (C.c_int, [_P, _P]),
    "tdpg_wirelength": (C.c_int, [_P, C.c_double, _P, _F64P, _F64P, _P]),
    "tdpg_set_grid": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_double]),
    "tdpg_density": (C.c_int, [_P, _F64P, _F64P, _P]),
    "tdpg_pp_set": (C.c_int, [_P, C.c_int64, _P, _P, _P]),
    "tdpg_pp_size": (C.c_int, [_P, _I64P]),
    "tdpg_pp_get": (C.c_int, [_P, _P, _P, _P]),
    "tdpg_pp_update": (C.c_int, [_P, C.c_int64, _P, _P, _P, C.c_double, C.c_double, C.c_double]),
    "tdpg_pp_loss": (C.c_int, [_P, C.c_int32, _F64P, _P]),
    "tdpg_objective": (C.c_int, [_P, C.c_double, C.c_double, C.c_double, C.c_int32, _P, _P, _P]),
    "tdpg_adam_step": (C.c_int, [C.c_int64, _P, _P, _P, _P, _I32P, C.c_double, C.c_double, C.c_double,
                                 C.c_double]),
    "tdpg_sta": (C.c_int, [_P, _P, _P, _P, _P, _P, _F64P, _F64P]),
    "tdpg_extract_endpoint": (C.c_int, [_P, C.c_int32, C.c_int32, _I64P]),
    "tdpg_paths_get": (C.c_int, [_P, _P, _P, _P]),
    "tdpg_paths_hits": (C.c_int, [_P, _I64P, _P, _P, _P]),
    "tdpg_last_timing_ms": (C.c_int, [_P, _F64P, _F64P]),
    "tdpg_place": (C.c_int, [_P, _P, _P, _P, _I32P, _I32P, _F64P]),
    "tdpg_engine_init": (C.c_int, [_P, _P, _P]),
    "tdpg_iterate_dev": (C.c_int, [_P, C.c_int32, _F64P]),
    "tdpg_engine_stats": (C.c_int, [_P, _I32P, _I32P, _I64P]),
    "tdpg_step_host": (C.c_int, [_P, _P, _P, _P]),
    "tdpg_set_pin_positions": (C.c_int, [_P, _P]),
    "tdpg_paths_counts": (C.c_int, [_P, _I64P]),
    "tdpg_set_core": (C.c_int, [_P, _P]),
    "tdpg_hpwl_pins": (C.c_int, [_P, _P, _F64P]),
    "tdpg_set_constraints": (C.c_int, [_P, C.c_double, C.c_double, C.c_double]),
    "tdpg_sta_fetch": (C.c_int, [_P, _P, _P, _P, _P, _P, _F64P, _F64P]),
    "tdpg_path_to": (C.c_int, [_P, C.c_int32, C.c_int32, _P, C.c_int32, _I32P, _F64P]),
    "tdpg_extract": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _I64P]),
    "tdpg_set_density_model": (C.c_int, [_P, C.c_int32]),
    "tdpg_density_fields": (C.c_int, [_P, _P, _P]),
    "tdpg_density_atomics": (C.c_int, [_P, _P]),
    "tdpg_partition_plan": (C.c_int, [C.c_int32, _P, C.c_int32, _P, _P]),
    "tdpg_set_partition": (C.c_int, [_P, C.c_int32, C.c_int32]),
    "tdpg_comm_unique_id": (C.c_int, [_P]),
    "tdpg_comm_init": (C.c_int, [_P, C.c_int32, C.c_int32, _P]),
    "tdpg_part_density": (C.c_int, [_P, _P, _I64P]),
    "tdpg_comm_bench": (C.c_int, [_P, C.c_int32, C.c_int64, _P]),
    "tdpg_part_step_a": (C.c_int, [_P, _P, _P, _I64P]),
    "tdpg_part_step_b": (C.c_int, [_P, _P]),
    "tdpg_paths_candidates": (C.c_int, [_P, _I64P]),
    "tdpg_k_worst": (C.c_int, [_P, C.c_int32, C.c_int32, _I32P, _P, _P, C.c_int32, _P]),
    "tdpg_set_round_callback": (C.c_int, [_P, _P, _P]),
    "tdpg_engine_times": (C.c_int, [_P, _F64P, _F64P, _I64P]),
    "tdpg_engine_paths": (C.c_int, [_P, _I64P, _I64P]),
    "tdpg_profile_iteration": (C.c_int, [_P, C.c_int32, _F64P, C.c_int32, C.c_char_p, C.c_int32]),
    "tdpg_generate": (C.c_int, [C.c_uint64, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                                C.c_double, C.c_int32, C.POINTER(_P)]),
    "tdpg_design_view": (C.c_int, [_P, _P, C.POINTER(_P)]),
    "tdpg_design_set_clock": (C.c_int, [_P, C.c_double]),
    "tdpg_design_destroy": (C.c_int, [_P]),
}


def lib():
    """Load the engine library; fails loudly when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `make -C paper_2503_11674_b200/csrc` "
                              "(the engine has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc):
    if rc:
        L = lib()
        _raise(rc, L.tdpg_last_error().decode())


def device_count():
    return lib().tdpg_device_count()


class Session:
    """One design resident on the GPU (the reference operator API, drop-in)."""

    def __init__(self, design: Design):
        self.lib = lib()
        self.d = design
        self._view = design.view()
        h = _P()
        _check(self.lib.tdpg_session_create(C.byref(self._view), C.byref(h)))
        self.h = h.value
        self.set_positions(design.positions)

    def close(self):
        if getattr(self, "h", None):
            self.lib.tdpg_session_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_constraints(self, clock_period, r_unit=None, c_unit=None):
        """DesignConstraints of the session (clock, RC units); the design copy follows."""
        r = self.d.r_unit if r_unit is None else r_unit
        c = self.d.c_unit if c_unit is None else c_unit
        _check(self.lib.tdpg_set_constraints(self.h, float(clock_period), float(r), float(c)))
        self.d = self.d.copy()  # (the caller's design object is left as it was)
        self.d.clock_period, self.d.r_unit, self.d.c_unit = float(clock_period), float(r), float(c)

    # positions -----------------------------------------------------------
    def set_positions(self, xy):
        xy = np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        _check(self.lib.tdpg_set_positions(self.h, xy.ctypes.data))

    def positions(self):
        out = np.zeros((self.d.n_cells, 2))
        _check(self.lib.tdpg_get_positions(self.h, out.ctypes.data))
        return out

    def _pos(self, xy):
        if xy is not None:
            self.set_positions(xy)

    def pin_positions(self, xy=None):
        self._pos(xy)
        out = np.zeros((self.d.n_pins, 2))
        _check(self.lib.tdpg_pin_positions(self.h, out.ctypes.data))
        return out

    # graph ---------------------------------------------------------------
    def graph(self):
        cnt = (C.c_int32 * 4)()
        level = np.zeros(self.d.n_pins, np.int32)
        _check(self.lib.tdpg_graph_info(self.h, cnt, level.ctypes.data))
        A = cnt[0] + cnt[1]
        arcs = [np.zeros(A, np.int32) for _ in range(4)]
        _check(self.lib.tdpg_graph_arcs(self.h, *[_p(a) for a in arcs]))
        return dict(n_net_arcs=cnt[0], n_cell_arcs=cnt[1], n_levels=cnt[2], level=level, arc_from=arcs[0],
                    arc_to=arcs[1], arc_kind=arcs[2], arc_owner=arcs[3])

    # objective terms -----------------------------------------------------
    def wirelength(self, gamma, xy=None, net_w=None, grad=True):
        self._pos(xy)
        wl, hp = C.c_double(), C.c_double()
        g = np.zeros((self.d.n_pins, 2)) if grad else None
        nw = None if net_w is None else np.ascontiguousarray(net_w, np.float64)
        _check(self.lib.tdpg_wirelength(self.h, gamma, _p(nw), C.byref(wl), C.byref(hp), _p(g)))
        return wl.value, hp.value, g

    def hpwl(self, xy=None):
        return self.wirelength(1.0, xy, grad=False)[1]

    def density(self, xy=None, nx=16, ny=16, td=0.6):
        self._pos(xy)
        _check(self.lib.tdpg_set_grid(self.h, nx, ny, td))
        v, o = C.c_double(), C.c_double()
        d = np.zeros((self.d.n_cells, 2))
        _check(self.lib.tdpg_density(self.h, C.byref(v), C.byref(o), d.ctypes.data))
        return v.value, o.value, d

    def set_density_model(self, model):
        """0 / "overflow": the reference's bin-overflow penalty; 1 / "electrostatic": DCT Poisson energy."""
        m = {"overflow": 0, "electrostatic": 1}.get(model, model)
        _check(self.lib.tdpg_set_density_model(self.h, int(m)))

    def density_atomics(self, nx, ny, td=0.6, xy=None):
        """(low-limb, upper-limb) shared-memory atomics of the density scatter at these positions."""
        self._pos(xy)
        _check(self.lib.tdpg_set_grid(self.h, nx, ny, td))
        out = np.zeros(2, np.int64)
        _check(self.lib.tdpg_density_atomics(self.h, out.ctypes.data))
        return int(out[0]), int(out[1])

    def density_fields(self, nx, ny):
        """Charge map and potential of the last electrostatic evaluation, shaped [nx, ny]."""
        rho, psi = np.zeros((nx, ny)), np.zeros((nx, ny))
        _check(self.lib.tdpg_density_fields(self.h, rho.ctypes.data, psi.ctypes.data))
        return rho, psi

    def set_ledger(self, ledger):
        if ledger is None or len(ledger[0]) == 0:
            _check(self.lib.tdpg_pp_set(self.h, 0, None, None, None))
            return
        a, b, w = (np.ascontiguousarray(ledger[0], np.int32), np.ascontiguousarray(ledger[1], np.int32),
                   np.ascontiguousarray(ledger[2], np.float64))
        _check(self.lib.tdpg_pp_set(self.h, a.size, _p(a), _p(b), _p(w)))

    def ledger(self):
        q = C.c_int64()
        _check(self.lib.tdpg_pp_size(self.h, C.byref(q)))
        out = (np.zeros(q.value, np.int32), np.zeros(q.value, np.int32), np.zeros(q.value))
        if q.value:
            _check(self.lib.tdpg_pp_get(self.h, *[_p(x) for x in out]))
        return out

    def pp_update(self, ledger, hits, wns, w0=10.0, w1=0.2):
        self.set_ledger(ledger)
        ha, hb, hs = (np.ascontiguousarray(hits[0], np.int32), np.ascontiguousarray(hits[1], np.int32),
                      np.ascontiguousarray(hits[2], np.float64))
        _check(self.lib.tdpg_pp_update(self.h, ha.size, _p(ha), _p(hb), _p(hs), wns, w0, w1))
        return self.ledger()

    def pp_loss_session(self, kind=0, ledger=None, xy=None):
        self._pos(xy)
        if ledger is not None:
            self.set_ledger(ledger)
        v = C.c_double()
        d = np.zeros((self.d.n_pins, 2))
        _check(self.lib.tdpg_pp_loss(self.h, kind, C.byref(v), d.ctypes.data))
        return v.value, d

    def objective(self, xy=None, nx=16, ny=16, td=0.6, gamma=1.0, lam=1.0, beta=0.0, kind=0, net_w=None,
                  ledger=None):
        self._pos(xy)
        _check(self.lib.tdpg_set_grid(self.h, nx, ny, td))
        self.set_ledger(ledger)
        nw = None if net_w is None else np.ascontiguousarray(net_w, np.float64)
        terms = np.zeros(6)
        d = np.zeros((self.d.n_cells, 2))
        _check(self.lib.tdpg_objective(self.h, gamma, lam, beta, kind, _p(nw), terms.ctypes.data, d.ctypes.data))
        return terms, d

    # timing ----------------------------------------------------------------
    def sta(self, xy=None):
        self._pos(xy)
        P = self.d.n_pins
        arr, req, slack = np.zeros(P), np.zeros(P), np.zeros(P)
        ak, rk = np.zeros(P, np.uint8), np.zeros(P, np.uint8)
        tns, wns = C.c_double(), C.c_double()
        _check(self.lib.tdpg_sta(self.h, arr.ctypes.data, req.ctypes.data, slack.ctypes.data, ak.ctypes.data,
                                 rk.ctypes.data, C.byref(tns), C.byref(wns)))
        return dict(arr=arr, req=req, slack=slack, arr_known=ak, req_known=rk, tns=tns.value, wns=wns.value)

    def extract(self, xy=None, n=0, k=1, run_sta=True, policy=0):
        """report_timing_endpoint(n, k) (policy 0) / report_timing(n) (policy 1, "topn"); n <= 0 = every
        violated endpoint."""
        if run_sta or xy is not None:
            self._pos(xy)
            tns, wns = C.c_double(), C.c_double()
            _check(self.lib.tdpg_sta(self.h, None, None, None, None, None, C.byref(tns), C.byref(wns)))
        cnt = (C.c_int64 * 5)()
        _check(self.lib.tdpg_extract(self.h, policy, n, k, cnt))
        return self._report(cnt)

    def k_worst(self, endpoint, k, xy=None):
        """k_worst_paths_to (paths.cpp:57-72): (paths, slacks); EndpointError for a non-endpoint."""
        if xy is not None:
            self._pos(xy)
        n = C.c_int32()
        cap = max(k, 1) * (self.d.n_pins + 1)
        start, pins, slack = np.zeros(k + 1, np.int32), np.zeros(cap, np.int32), np.zeros(max(k, 1))
        _check(self.lib.tdpg_k_worst(self.h, endpoint, k, C.byref(n), start.ctypes.data, pins.ctypes.data, cap,
                                     slack.ctypes.data))
        return [pins[start[i]:start[i + 1]].tolist() for i in range(n.value)], slack[:n.value]

    # partitioned multi-GPU mode -------------------------------
    def set_partition(self, rank, world):
        _check(self.lib.tdpg_set_partition(self.h, rank, world))

    def comm_init(self, rank, world, uid: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(self.lib.tdpg_comm_init(self.h, rank, world, buf))

    def comm_bench(self, iters=20):
        """Device ms of the partitioned iteration's two all-reduces alone: (density grid, gradient buffer)."""
        ms = (C.c_double * 2)()
        _check(self.lib.tdpg_comm_bench(self.h, iters, red_size(self), ms))
        return ms[0], ms[1]

    def part_density_into(self, out: np.ndarray):
        """Split phase 0: this rank's density scatter; its int64 grid into `out` (returns the bin count)."""
        n = C.c_int64()
        _check(self.lib.tdpg_part_density(self.h, out.ctypes.data if out is not None else None, C.byref(n)))
        return n.value

    def part_step_a_into(self, acc_total: np.ndarray, out: np.ndarray):
        """Split phase A: the grid summed over ranks in, this rank's all-reduce buffer out (returns its size)."""
        acc_total = np.ascontiguousarray(acc_total, np.int64)
        n = C.c_int64()
        _check(self.lib.tdpg_part_step_a(self.h, acc_total.ctypes.data, out.ctypes.data if out is not None else None,
                                         C.byref(n)))
        return n.value

    def part_step_b(self, red: np.ndarray):
        red = np.ascontiguousarray(red, np.float64)
        _check(self.lib.tdpg_part_step_b(self.h, red.ctypes.data))

    def path_to(self, pin, rank=0):
        """PathEnumerator::path_to(pin, rank): (pins, delay) or None once exhausted."""
        buf = np.zeros(self.d.n_pins + 1, np.int32)
        n, dl = C.c_int32(), C.c_double()
        _check(self.lib.tdpg_path_to(self.h, pin, rank, buf.ctypes.data, buf.size, C.byref(n), C.byref(dl)))
        return (buf[:n.value].tolist(), dl.value) if n.value else None

    def _report(self, cnt):
        npath, total = cnt[0], cnt[1]
        start = np.zeros(npath + 1, np.int32)
        pins = np.zeros(max(total, 1), np.int32)
        slack = np.zeros(max(npath, 1))
        _check(self.lib.tdpg_paths_get(self.h, start.ctypes.data, pins.ctypes.data, slack.ctypes.data))
        nh = C.c_int64()
        _check(self.lib.tdpg_paths_hits(self.h, C.byref(nh), None, None, None))
        m = max(nh.value, 1)
        ha, hb, hs = np.zeros(m, np.int32), np.zeros(m, np.int32), np.zeros(m)
        _check(self.lib.tdpg_paths_hits(self.h, C.byref(nh), ha.ctypes.data, hb.ctypes.data, hs.ctypes.data))
        sta_ms, ex_ms = C.c_double(), C.c_double()
        _check(self.lib.tdpg_last_timing_ms(self.h, C.byref(sta_ms), C.byref(ex_ms)))
        return dict(start=start, pins=pins[:total], slack=slack[:npath], n_paths=npath, unique_endpoints=cnt[2],
                    unique_pin_pairs=cnt[3], candidates_generated=cnt[4],
                    hits=(ha[:nh.value], hb[:nh.value], hs[:nh.value]), sta_ms=sta_ms.value, extract_ms=ex_ms.value)

    # placement -------------------------------------------------------------
    def place(self, cfg: dict | None = None, xy=None):
        c = make_config(cfg)
        self._pos(xy if xy is not None else self.d.positions)
        rows = (TdpgTraceRow * max(c.max_iters, 1))()
        nr, so = C.c_int32(), C.c_int32()
        fin = (C.c_double * 3)()
        _check(self.lib.tdpg_place(self.h, C.byref(c), self.d.pos_explicit.ctypes.data, rows, C.byref(nr),
                                   C.byref(so), fin))
        return dict(positions=self.positions(), trace=[rows[i] for i in range(nr.value)], iterations=nr.value,
                    stop_reason="overflow" if so.value else "max_iters", tns=fin[0], wns=fin[1], hpwl=fin[2],
                    ledger=self.ledger())

    def place_host(self, cfg: dict, xy_in_ptr: int, xy_out_ptr: int):
        """run_placement through the C-ABI with caller-owned host buffers (e.g. pinned): positions in,
        the whole device loop (tdpg_place), positions and trace out.  Returns (rows, final tns/wns/hpwl)."""
        c = make_config(cfg)
        rows = (TdpgTraceRow * max(c.max_iters, 1))()
        nr, so = C.c_int32(), C.c_int32()
        fin = (C.c_double * 3)()
        _check(self.lib.tdpg_set_positions(self.h, C.c_void_p(xy_in_ptr)))
        _check(self.lib.tdpg_place(self.h, C.byref(c), self.d.pos_explicit.ctypes.data, rows, C.byref(nr),
                                   C.byref(so), fin))
        _check(self.lib.tdpg_get_positions(self.h, C.c_void_p(xy_out_ptr)))
        return nr.value, tuple(fin)

    def engine_init(self, cfg: dict | None = None, xy=None):
        c = make_config(cfg)
        self._pos(xy if xy is not None else self.d.positions)
        self._cfg = c
        _check(self.lib.tdpg_engine_init(self.h, C.byref(c), self.d.pos_explicit.ctypes.data))

    def iterate(self, n):
        ms = C.c_double()
        _check(self.lib.tdpg_iterate_dev(self.h, n, C.byref(ms)))
        return ms.value

    def step_host(self, xy_in_ptr, xy_out_ptr):
        """One iteration through host buffers (raw pointers, e.g. pinned memory)."""
        row = TdpgTraceRow()
        _check(self.lib.tdpg_step_host(self.h, xy_in_ptr, xy_out_ptr, C.byref(row)))
        return row

    def engine_stats(self):
        it, rf, ln = C.c_int32(), C.c_int32(), C.c_int64()
        _check(self.lib.tdpg_engine_stats(self.h, C.byref(it), C.byref(rf), C.byref(ln)))
        tot, last, q = C.c_double(), C.c_double(), C.c_int64()
        _check(self.lib.tdpg_engine_times(self.h, C.byref(tot), C.byref(last), C.byref(q)))
        pa, pp = C.c_int64(), C.c_int64()
        _check(self.lib.tdpg_engine_paths(self.h, C.byref(pa), C.byref(pp)))
        return dict(iterations=it.value, refreshes=rf.value, kernel_launches=ln.value, refresh_ms=tot.value,
                    last_refresh_ms=last.value, ledger_pairs=q.value, paths=pa.value, path_pins=pp.value)

    def profile_iteration(self, reps=5):
        n = 16
        out = (C.c_double * n)()
        names = C.create_string_buffer(n * 32)
        _check(self.lib.tdpg_profile_iteration(self.h, reps, out, n, names, 32))
        res = {}
        for i in range(n):
            nm = names.raw[i * 32:(i + 1) * 32].split(b"\0")[0].decode()
            if nm:
                res[nm] = out[i]
        return res

    # stateless helpers (tiny one-net designs on the device) ---------------------
    @staticmethod
    def _one_net_design(xy):
        xy = np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        n = xy.shape[0]
        return Design(cell_w=np.zeros(0), cell_h=np.zeros(0), cell_delay=np.zeros(0), cell_fixed=np.zeros(0),
                      pin_cell=-np.ones(n), pin_term=xy, pin_off=np.zeros((n, 2)),
                      pin_dir=[1] + [0] * (n - 1), pin_cap=np.zeros(n), net_start=[0, n] if n >= 2 else [0],
                      net_pins=list(range(n)) if n >= 2 else [], sources=[], endpoints=[], clock_period=1.0,
                      r_unit=1.0, c_unit=1.0, core=(0.0, 0.0, 1.0, 1.0), positions=np.zeros((0, 2)),
                      pos_explicit=np.zeros(0))

    @classmethod
    def wa(cls, xy, gamma):
        """wa_wirelength on one net (wirelength.cpp:49-58), computed by the device kernel."""
        xy = np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        if xy.shape[0] < 2:
            return 0.0, np.zeros_like(xy)
        s = cls(cls._one_net_design(xy))
        v, _, g = s.wirelength(gamma)
        return v, g

    @classmethod
    def pp_loss(cls, ledger, pin_xy, kind=0):
        """pin_pair_loss (pin_pairs.cpp:17-49), computed by the device kernel."""
        s = cls(cls._one_net_design(pin_xy))
        return s.pp_loss_session(kind, ledger)

    @classmethod
    def adam_step(cls, x, g, m, v, t, lr, b1=0.9, b2=0.999, eps=1e-8):
        tt = C.c_int32(t)
        _check(lib().tdpg_adam_step(x.size, x.ctypes.data, g.ctypes.data, m.ctypes.data, v.ctypes.data, C.byref(tt),
                                    lr, b1, b2, eps))
        return tt.value


def comm_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0 creates it, every rank passes it to Session.comm_init)."""
    buf = (C.c_uint8 * 128)()
    _check(lib().tdpg_comm_unique_id(buf))
    return bytes(buf)


def partition_plan(net_start, world):
    """Per-rank WA block ranges [bounds[r], bounds[r+1]) and their net-pin entry counts (host only)."""
    ns = np.ascontiguousarray(net_start, np.int32)
    bounds = np.zeros(world + 1, np.int32)
    ent = np.zeros(world, np.int64)
    _check(lib().tdpg_partition_plan(ns.size - 1, ns.ctypes.data, world, bounds.ctypes.data, ent.ctypes.data))
    return bounds, ent


def red_size(session) -> int:
    """Length of the partitioned engine's all-reduce buffer (2C + 3 WA blocks)."""
    return 2 * session.d.n_cells + 3 * int(partition_plan(session.d.net_start, 1)[0][1])


def generate(seed=1, cells=100, registers=-1, fanout=2.0, fail_frac=0.2, r_unit=1e-4, c_unit=1e-4,
             calibrate=True) -> Design:
    """generate_synthetic (generator.cpp:60-263): same netlist as the reference, O(N log N);
    the clock calibration's coarse placement runs on the GPU (calibrate=False keeps clock 1.0)."""
    L = lib()
    h = _P()
    _check(L.tdpg_generate(seed, cells, registers, fanout, fail_frac, r_unit, c_unit, int(calibrate), C.byref(h)))
    try:
        v = TdpgNetlist()
        pos = _P()
        _check(L.tdpg_design_view(h, C.byref(v), C.byref(pos)))

        def arr(ptr, n, ct, shape=None):
            if n == 0:
                return np.zeros(shape or (0,), dtype=np.dtype(ct))
            a = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).copy()
            return a.reshape(shape) if shape else a

        Cn, P, N = v.n_cells, v.n_pins, v.n_nets
        E = arr(v.net_start, N + 1, C.c_int32)[-1]
        d = Design(cell_w=arr(v.cell_w, Cn, C.c_double), cell_h=arr(v.cell_h, Cn, C.c_double),
                   cell_delay=arr(v.cell_delay, Cn, C.c_double), cell_fixed=arr(v.cell_fixed, Cn, C.c_uint8),
                   pin_cell=arr(v.pin_cell, P, C.c_int32), pin_term=arr(v.pin_term, 2 * P, C.c_double, (P, 2)),
                   pin_off=arr(v.pin_off, 2 * P, C.c_double, (P, 2)), pin_dir=arr(v.pin_dir, P, C.c_uint8),
                   pin_cap=arr(v.pin_cap, P, C.c_double), net_start=arr(v.net_start, N + 1, C.c_int32),
                   net_pins=arr(v.net_pins, int(E), C.c_int32), sources=arr(v.sources, v.n_sources, C.c_int32),
                   endpoints=arr(v.endpoints, v.n_endpoints, C.c_int32), clock_period=v.clock_period,
                   r_unit=v.r_unit, c_unit=v.c_unit, core=tuple(v.core),
                   positions=arr(pos.value, 2 * Cn, C.c_double, (Cn, 2)), pos_explicit=np.zeros(Cn, np.uint8))
        return d
    finally:
        L.tdpg_design_destroy(h)


def design_bin_write(d: Design, path: str) -> None:
    """tdpg_design_bin_write: the binary design file through the C-ABI (same bytes as design.save_bin)."""
    v = d.view()
    _check(lib().tdpg_design_bin_write(path.encode(), C.byref(v), d.positions.ctypes.data, d.pos_explicit.ctypes.data,
                                       float(d.default_cell_delay)))


def design_bin_read(path: str) -> Design:
    """tdpg_design_bin_info + tdpg_design_bin_read into numpy arrays (the C-ABI reader)."""
    L = lib()
    cnt = np.zeros(6, np.int64)
    names = C.c_int32()
    _check(L.tdpg_design_bin_info(path.encode(), cnt.ctypes.data, C.byref(names)))
    Cn, P, N, E, S, EP = (int(x) for x in cnt)
    a = dict(cell_w=np.zeros(Cn), cell_h=np.zeros(Cn), cell_delay=np.zeros(Cn), cell_fixed=np.zeros(Cn, np.uint8),
             pin_cell=np.zeros(P, np.int32), pin_term=np.zeros((P, 2)), pin_off=np.zeros((P, 2)),
             pin_dir=np.zeros(P, np.uint8), pin_cap=np.zeros(P), net_start=np.zeros(N + 1, np.int32),
             net_pins=np.zeros(E, np.int32), sources=np.zeros(S, np.int32), endpoints=np.zeros(EP, np.int32))
    v = TdpgNetlist()
    v.n_cells, v.n_pins, v.n_nets, v.n_sources, v.n_endpoints = Cn, P, N, S, EP
    for k, x in a.items():
        setattr(v, k, x.ctypes.data)
    pos, expl = np.zeros((Cn, 2)), np.zeros(Cn, np.uint8)
    cap = 0
    blob = None
    if names.value:
        import os
        cap = os.path.getsize(path)
        blob = C.create_string_buffer(cap)
    _check(L.tdpg_design_bin_read(path.encode(), C.byref(v), pos.ctypes.data, expl.ctypes.data,
                                  C.cast(blob, C.c_void_p) if blob is not None else None, cap))
    pin_names = None
    if blob is not None:
        pin_names = [s.decode() for s in blob.raw.split(b"\0")[:P]]
    with open(path, "rb") as f:  # (default cell delay: header slot 7)
        f.seek(64 + 7 * 8)
        dcd = float(np.frombuffer(f.read(8), "<f8")[0])
    return Design(clock_period=v.clock_period, r_unit=v.r_unit, c_unit=v.c_unit, core=tuple(v.core),
                  positions=pos, pos_explicit=expl, pin_names=pin_names, default_cell_delay=dcd, **a)
