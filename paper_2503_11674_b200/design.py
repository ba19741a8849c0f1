"""Flat, numpy-backed design container mirroring ``tdp::Design``.

The reference holds a design as ``Netlist`` (cells, pins, nets, sources,
endpoints) + ``DesignConstraints`` + per-cell positions
(``/root/reference/proj/include/tdp/netlist.hpp:11-93``).  Here the same data
is a structure of arrays, which is exactly what the C-ABI
(``include/tdpg.h::tdpg_netlist``) and the GPU session upload.  The JSON schema
is the reference's (``proj/include/tdp/design_io.hpp:10-17``,
``proj/src/design_io.cpp:63-193``).
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np


class TdpgNetlist(C.Structure):
    """ctypes twin of ``tdpg_netlist`` (include/tdpg.h)."""

    _fields_ = [
        ("n_cells", C.c_int32),
        ("n_pins", C.c_int32),
        ("n_nets", C.c_int32),
        ("n_sources", C.c_int32),
        ("n_endpoints", C.c_int32),
        ("cell_w", C.c_void_p),
        ("cell_h", C.c_void_p),
        ("cell_delay", C.c_void_p),
        ("cell_fixed", C.c_void_p),
        ("pin_cell", C.c_void_p),
        ("pin_term", C.c_void_p),
        ("pin_off", C.c_void_p),
        ("pin_dir", C.c_void_p),
        ("pin_cap", C.c_void_p),
        ("net_start", C.c_void_p),
        ("net_pins", C.c_void_p),
        ("sources", C.c_void_p),
        ("endpoints", C.c_void_p),
        ("clock_period", C.c_double),
        ("r_unit", C.c_double),
        ("c_unit", C.c_double),
        ("core", C.c_double * 4),
        ("pin_names", C.c_void_p),
    ]


class TdpgConfig(C.Structure):
    """ctypes twin of ``tdpg_config`` == ``tdp::OptimizerConfig`` (placer.hpp:22-57)."""

    _fields_ = [
        ("gamma_frac", C.c_double),
        ("grid_nx", C.c_int32),
        ("grid_ny", C.c_int32),
        ("target_density", C.c_double),
        ("beta", C.c_double),
        ("pp_loss", C.c_int32),
        ("net_weighting", C.c_int32),
        ("m", C.c_int32),
        ("w0", C.c_double),
        ("w1", C.c_double),
        ("timing_start_iter", C.c_int32),
        ("extraction", C.c_int32),
        ("k", C.c_int32),
        ("max_iters", C.c_int32),
        ("stop_overflow", C.c_double),
        ("mu", C.c_double),
        ("lambda0", C.c_double),
        ("lambda_max", C.c_double),
        ("step0_frac", C.c_double),
        ("step_decay", C.c_double),
        ("adam_beta1", C.c_double),
        ("adam_beta2", C.c_double),
        ("adam_eps", C.c_double),
        ("seed", C.c_uint64),
        ("init_jitter_frac", C.c_double),
        ("threads", C.c_int32),
        ("density_model", C.c_int32),  # extension: "overflow" (the reference) | "electrostatic"
    ]


class TdpgTraceRow(C.Structure):
    _fields_ = [
        ("iter", C.c_int32),
        ("has_timing", C.c_int32),
        ("hpwl", C.c_double),
        ("overflow", C.c_double),
        ("tns", C.c_double),
        ("wns", C.c_double),
        ("wl_term", C.c_double),
        ("density_term", C.c_double),
        ("pp_term", C.c_double),
        ("lambda_", C.c_double),
        ("beta_pp", C.c_double),
    ]


# OptimizerConfig defaults (proj/include/tdp/placer.hpp:22-57).
CONFIG_DEFAULTS = {
    "name": "default",
    "gamma_frac": 0.01,
    "grid_nx": 16,
    "grid_ny": 16,
    "target_density": 0.6,
    "beta": 2.5e-5,
    "pp_loss": "quadratic",
    "net_weighting": False,
    "m": 15,
    "w0": 10.0,
    "w1": 0.2,
    "timing_start_iter": 500,
    "extraction": "endpoint",
    "k": 1,
    "max_iters": 1500,
    "stop_overflow": 0.0,
    "mu": 1.05,
    "lambda0": "auto",
    "lambda_max": 1e8,
    "step0_frac": 0.01,
    "step_decay": 0.999,
    "adam_beta1": 0.9,
    "adam_beta2": 0.999,
    "adam_eps": 1e-8,
    "seed": 1,
    "init_jitter_frac": 0.02,
    "threads": 1,
    "density_model": "overflow",  # extension (not a reference key): "overflow" | "electrostatic"
}


def make_config(cfg: dict | None = None) -> TdpgConfig:
    """Resolve a reference-schema config dict into a ``TdpgConfig``."""
    c = dict(CONFIG_DEFAULTS)
    for k, v in (cfg or {}).items():
        if k not in c:
            raise ValueError(f'parse error: config: unknown key "{k}"')
        c[k] = v
    out = TdpgConfig()
    for name, _ in TdpgConfig._fields_:
        v = c[name]
        if name == "pp_loss":
            v = {"quadratic": 0, "linear": 1}[v]
        elif name == "extraction":
            v = {"endpoint": 0, "topn": 1}[v]
        elif name == "density_model":
            v = {"overflow": 0, "electrostatic": 1}[v]
        elif name == "lambda0":
            v = 0.0 if v == "auto" else float(v)
        elif name == "net_weighting":
            v = int(bool(v))
        setattr(out, name, v)
    return out


def _f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a.reshape(shape) if shape is not None else a


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _u8(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8))


@dataclass
class Design:
    """SoA twin of ``tdp::Design``; ids are array indices as in the reference."""

    cell_w: np.ndarray
    cell_h: np.ndarray
    cell_delay: np.ndarray
    cell_fixed: np.ndarray
    pin_cell: np.ndarray
    pin_term: np.ndarray  # [P, 2]
    pin_off: np.ndarray  # [P, 2]
    pin_dir: np.ndarray  # 0 in, 1 out
    pin_cap: np.ndarray
    net_start: np.ndarray
    net_pins: np.ndarray
    sources: np.ndarray
    endpoints: np.ndarray
    clock_period: float
    r_unit: float
    c_unit: float
    core: tuple
    positions: np.ndarray  # [C, 2] lower-left origins
    pos_explicit: np.ndarray
    cell_names: list | None = None
    pin_names: list | None = None
    net_names: list | None = None
    default_cell_delay: float = 1.0
    _keep: list = field(default_factory=list, repr=False)

    def __post_init__(self):
        self.cell_w = _f64(self.cell_w)
        self.cell_h = _f64(self.cell_h)
        self.cell_delay = _f64(self.cell_delay)
        self.cell_fixed = _u8(self.cell_fixed)
        self.pin_cell = _i32(self.pin_cell)
        self.pin_term = _f64(self.pin_term, (-1, 2))
        self.pin_off = _f64(self.pin_off, (-1, 2))
        self.pin_dir = _u8(self.pin_dir)
        self.pin_cap = _f64(self.pin_cap)
        self.net_start = _i32(self.net_start)
        self.net_pins = _i32(self.net_pins)
        self.sources = _i32(self.sources)
        self.endpoints = _i32(self.endpoints)
        self.positions = _f64(self.positions, (-1, 2))
        self.pos_explicit = _u8(self.pos_explicit)
        self.core = tuple(float(v) for v in self.core)

    # ---- sizes -------------------------------------------------------------
    @property
    def n_cells(self):
        return int(self.cell_w.shape[0])

    @property
    def n_pins(self):
        return int(self.pin_cell.shape[0])

    @property
    def n_nets(self):
        return int(self.net_start.shape[0]) - 1

    @property
    def n_net_pins(self):
        return int(self.net_start[-1])

    def counts(self):
        return dict(cells=self.n_cells, pins=self.n_pins, nets=self.n_nets, net_pins=self.n_net_pins,
                    sources=int(self.sources.size), endpoints=int(self.endpoints.size))

    # ---- C view ------------------------------------------------------------
    def view(self) -> TdpgNetlist:
        v = TdpgNetlist()
        v.n_cells, v.n_pins, v.n_nets = self.n_cells, self.n_pins, self.n_nets
        v.n_sources, v.n_endpoints = int(self.sources.size), int(self.endpoints.size)
        for name in ("cell_w", "cell_h", "cell_delay", "cell_fixed", "pin_cell", "pin_term", "pin_off",
                     "pin_dir", "pin_cap", "net_start", "net_pins", "sources", "endpoints"):
            setattr(v, name, getattr(self, name).ctypes.data)
        v.clock_period, v.r_unit, v.c_unit = float(self.clock_period), float(self.r_unit), float(self.c_unit)
        v.core[:] = self.core
        v.pin_names = None
        if self.pin_names is not None:
            arr = (C.c_char_p * self.n_pins)(*[n.encode() for n in self.pin_names])
            self._keep = [arr]
            v.pin_names = C.cast(arr, C.c_void_p).value
        return v

    def copy(self) -> "Design":
        kw = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in self.__dict__.items() if k != "_keep"}
        return Design(**kw)

    # ---- geometry helpers ----------------------------------------------------
    @property
    def span(self):
        w, h = self.core[2] - self.core[0], self.core[3] - self.core[1]
        return w if w > h else h

    def net_pin_lists(self):
        return [self.net_pins[self.net_start[e]:self.net_start[e + 1]] for e in range(self.n_nets)]

    # ---- reference JSON schema (design_io.cpp) ------------------------------
    @classmethod
    def from_json(cls, obj) -> "Design":
        """Parse the reference design schema (proj/src/design_io.cpp:63-193).

        Structural checks mirror the reference's messages; full semantic
        validation (validate_design, design_io.cpp:195-256) is ``validate``.
        """
        if isinstance(obj, (str, bytes)):
            try:
                obj = json.loads(obj)
            except json.JSONDecodeError as e:
                raise ValueError(f"parse error: {e}") from None
        if not isinstance(obj, dict):
            raise ValueError("parse error: top level must be an object")
        allowed = {"core", "clock_period", "r_unit", "c_unit", "default_cell_delay", "cells", "pins", "nets",
                   "sources", "endpoints"}
        for k in obj:
            if k not in allowed:
                raise ValueError(f'parse error: design: unknown key "{k}"')
        for k in ("core", "clock_period", "r_unit", "c_unit", "cells", "pins", "nets", "sources", "endpoints"):
            if k not in obj:
                raise ValueError(f'parse error: design: missing "{k}"')
        core = obj["core"]
        if not (isinstance(core, list) and len(core) == 4):
            raise ValueError("parse error: core must be [x_lo, y_lo, x_hi, y_hi]")
        dcd = float(obj.get("default_cell_delay", 1.0))
        cells = obj["cells"]
        cid = {}
        cw, ch, cd, cf, pos, expl, cnames = [], [], [], [], [], [], []
        for c in cells:
            name = c["name"]
            if name in cid:
                raise ValueError(f'validation error: duplicate cell name "{name}"')
            cid[name] = len(cnames)
            cnames.append(name)
            cw.append(float(c["width"]))
            ch.append(float(c["height"]))
            cd.append(float(c.get("delay", dcd)))
            cf.append(1 if c.get("fixed", False) else 0)
            if ("x" in c) != ("y" in c):
                raise ValueError(f'parse error: cell "{name}": x and y must be given together')
            has = "x" in c
            expl.append(1 if has else 0)
            pos.append((float(c["x"]), float(c["y"])) if has else (0.0, 0.0))
        pid = {}
        pc, pt, po, pd, pcap, pnames = [], [], [], [], [], []
        for p in obj["pins"]:
            name = p["name"]
            if name in pid:
                raise ValueError(f'validation error: duplicate pin name "{name}"')
            if ("cell" in p) == ("terminal" in p):
                raise ValueError(f'parse error: pin "{name}": exactly one of "cell" or "terminal" required')
            pid[name] = len(pnames)
            pnames.append(name)
            if "cell" in p:
                if p["cell"] not in cid:
                    raise ValueError(f'validation error: pin "{name}": unknown cell "{p["cell"]}"')
                pc.append(cid[p["cell"]])
                pt.append((0.0, 0.0))
            else:
                pc.append(-1)
                pt.append((float(p["terminal"]["x"]), float(p["terminal"]["y"])))
            po.append((float(p.get("dx", 0.0)), float(p.get("dy", 0.0))))
            if p["dir"] not in ("in", "out"):
                raise ValueError(f'parse error: pin "{name}": dir must be "in" or "out"')
            pd.append(1 if p["dir"] == "out" else 0)
            pcap.append(float(p.get("cap", 0.0)))

        def look(n, where):
            if n not in pid:
                raise ValueError(f'validation error: {where}: unknown pin "{n}"')
            return pid[n]

        ns, npins, nnames = [0], [], []
        for n in obj["nets"]:
            where = f'net "{n["name"]}"'
            nnames.append(n["name"])
            npins.append(look(n["driver"], where))
            for s in n["sinks"]:
                npins.append(look(s, where))
            ns.append(len(npins))
        src = [look(s, "sources") for s in obj["sources"]]
        eps = [look(e, "endpoints") for e in obj["endpoints"]]
        x0, y0, x1, y1 = (float(v) for v in core)
        for c in range(len(cnames)):
            if not expl[c]:
                pos[c] = ((x0 + x1) / 2.0 - cw[c] / 2.0, (y0 + y1) / 2.0 - ch[c] / 2.0)
        d = cls(cell_w=cw, cell_h=ch, cell_delay=cd, cell_fixed=cf, pin_cell=pc,
                pin_term=np.asarray(pt, dtype=np.float64).reshape(-1, 2),
                pin_off=np.asarray(po, dtype=np.float64).reshape(-1, 2), pin_dir=pd, pin_cap=pcap,
                net_start=ns, net_pins=npins, sources=src, endpoints=eps,
                clock_period=float(obj["clock_period"]), r_unit=float(obj["r_unit"]), c_unit=float(obj["c_unit"]),
                core=(x0, y0, x1, y1), positions=np.asarray(pos, dtype=np.float64).reshape(-1, 2),
                pos_explicit=expl, cell_names=cnames, pin_names=pnames, net_names=nnames,
                default_cell_delay=dcd)
        d.validate()
        return d

    def validate(self):
        """validate_design (proj/src/design_io.cpp:195-256), same messages."""
        x0, y0, x1, y1 = self.core
        if not (x1 > x0 and y1 > y0):
            raise ValueError("validation error: core region is degenerate")
        if not self.clock_period > 0.0:
            raise ValueError("validation error: clock_period must be > 0")
        if not (self.r_unit > 0.0) or not (self.c_unit > 0.0):
            raise ValueError("validation error: r_unit and c_unit must be > 0")
        cn = self.cell_names or [f"c{i}" for i in range(self.n_cells)]
        pn = self.pin_names or [f"p{i}" for i in range(self.n_pins)]
        nn = self.net_names or [f"n{i}" for i in range(self.n_nets)]
        any_movable = False
        for c in range(self.n_cells):
            w, h = self.cell_w[c], self.cell_h[c]
            if not (w > 0.0) or not (h > 0.0):
                raise ValueError(f'validation error: zero-size cell "{cn[c]}"')
            if w > x1 - x0 or h > y1 - y0:
                raise ValueError(f'validation error: cell "{cn[c]}" larger than core')
            if self.cell_fixed[c]:
                if not self.pos_explicit[c]:
                    raise ValueError(f'validation error: fixed cell "{cn[c]}" has no coordinates')
                px, py = self.positions[c]
                if not (px >= x0 and py >= y0 and px + w <= x1 and py + h <= y1):
                    raise ValueError(f'validation error: fixed cell "{cn[c]}" outside core')
            else:
                any_movable = True
        if not any_movable:
            raise ValueError("validation error: no movable cells")
        bad = np.nonzero(self.pin_cap < 0.0)[0]
        if bad.size:
            raise ValueError(f'validation error: pin "{pn[bad[0]]}": cap must be >= 0')
        owner = np.full(self.n_pins, -1, dtype=np.int64)
        for e in range(self.n_nets):
            s0, s1 = self.net_start[e], self.net_start[e + 1]
            drv = self.net_pins[s0]
            where = f'net "{nn[e]}"'
            if self.pin_dir[drv] != 1:
                raise ValueError(f"validation error: {where}: driver must be an output pin")
            if s1 - s0 < 2:
                raise ValueError(f"validation error: {where}: needs at least one sink")
            for i in range(s0, s1):
                p = self.net_pins[i]
                if i > s0:
                    if p == drv:
                        raise ValueError(f"validation error: {where}: driver and sink on the same pin")
                    if self.pin_dir[p] != 0:
                        raise ValueError(f'validation error: {where}: sink "{pn[p]}" must be an input pin')
                if owner[p] >= 0:
                    raise ValueError(f'validation error: pin "{pn[p]}" used by nets "{nn[owner[p]]}" and "{nn[e]}"')
                owner[p] = e
        for s in self.sources:
            if self.pin_dir[s] != 1:
                raise ValueError(f'validation error: source pin "{pn[s]}" must be an output')
        for e in self.endpoints:
            if self.pin_dir[e] != 0:
                raise ValueError(f'validation error: endpoint pin "{pn[e]}" must be an input')

    def to_json_obj(self) -> dict:
        cn = self.cell_names or [f"c{i}" for i in range(self.n_cells)]
        pn = self.pin_names or [f"p{i}" for i in range(self.n_pins)]
        nn = self.net_names or [f"n{i}" for i in range(self.n_nets)]
        cells = []
        for c in range(self.n_cells):
            jc = {"name": cn[c], "width": float(self.cell_w[c]), "height": float(self.cell_h[c])}
            if self.cell_fixed[c]:
                jc["fixed"] = True
            if self.pos_explicit[c]:
                jc["x"], jc["y"] = float(self.positions[c, 0]), float(self.positions[c, 1])
            if self.cell_delay[c] != self.default_cell_delay:
                jc["delay"] = float(self.cell_delay[c])
            cells.append(jc)
        pins = []
        for p in range(self.n_pins):
            jp = {"name": pn[p]}
            if self.pin_cell[p] < 0:
                jp["terminal"] = {"x": float(self.pin_term[p, 0]), "y": float(self.pin_term[p, 1])}
            else:
                jp["cell"] = cn[self.pin_cell[p]]
            if self.pin_off[p, 0] != 0.0:
                jp["dx"] = float(self.pin_off[p, 0])
            if self.pin_off[p, 1] != 0.0:
                jp["dy"] = float(self.pin_off[p, 1])
            jp["dir"] = "out" if self.pin_dir[p] else "in"
            if self.pin_cap[p] != 0.0:
                jp["cap"] = float(self.pin_cap[p])
            pins.append(jp)
        nets = []
        for e in range(self.n_nets):
            s0, s1 = self.net_start[e], self.net_start[e + 1]
            nets.append({"name": nn[e], "driver": pn[self.net_pins[s0]],
                         "sinks": [pn[p] for p in self.net_pins[s0 + 1:s1]]})
        return {"core": list(self.core), "clock_period": float(self.clock_period), "r_unit": float(self.r_unit),
                "c_unit": float(self.c_unit), "default_cell_delay": float(self.default_cell_delay),
                "cells": cells, "pins": pins, "nets": nets,
                "sources": [pn[s] for s in self.sources], "endpoints": [pn[e] for e in self.endpoints]}

    # ---- binary format (for >= 200K designs; JSON is ~0.84 GB at 1M) ---------
    _ARRAYS = ("cell_w", "cell_h", "cell_delay", "cell_fixed", "pin_cell", "pin_term", "pin_off", "pin_dir",
               "pin_cap", "net_start", "net_pins", "sources", "endpoints", "positions", "pos_explicit")

    def save_npz(self, path):
        np.savez(path, clock=np.array([self.clock_period, self.r_unit, self.c_unit]), core=np.array(self.core),
                 **{k: getattr(self, k) for k in self._ARRAYS})

    @classmethod
    def load_npz(cls, path) -> "Design":
        z = np.load(path)
        clk = z["clock"]
        return cls(**{k: z[k] for k in cls._ARRAYS}, clock_period=float(clk[0]), r_unit=float(clk[1]),
                   c_unit=float(clk[2]), core=tuple(z["core"]))


# ---- binary design file (SoA, scalable; the reference's JSON schema does not scale to 1M cells) ----------
# Layout (little-endian; every section starts 8-byte aligned; mirrored by csrc/design_io.cu):
#   0   char[8] "TDPGDSN1" | u32 version (1) | u32 flags (bit 0: pin names present)
#   16  i64 n_cells, n_pins, n_nets, n_net_pins, n_sources, n_endpoints
#   64  f64 clock_period, r_unit, c_unit, core[4], default_cell_delay
#   128 cell_w f64[C] | cell_h f64[C] | cell_delay f64[C] | positions f64[2C] | pin_term f64[2P] |
#       pin_off f64[2P] | pin_cap f64[P] | pin_cell i32[P] | net_start i32[N+1] | net_pins i32[E] |
#       sources i32[S] | endpoints i32[EP] | cell_fixed u8[C] | pos_explicit u8[C] | pin_dir u8[P] |
#       [flags & 1] u64 byte count + the pin names, each NUL-terminated
BIN_MAGIC = b"TDPGDSN1"
BIN_HEADER = 128


def _bin_sections(c):
    C, P, N, E, S, EP = c
    return [("cell_w", np.float64, (C,)), ("cell_h", np.float64, (C,)), ("cell_delay", np.float64, (C,)),
            ("positions", np.float64, (C, 2)), ("pin_term", np.float64, (P, 2)), ("pin_off", np.float64, (P, 2)),
            ("pin_cap", np.float64, (P,)), ("pin_cell", np.int32, (P,)), ("net_start", np.int32, (N + 1,)),
            ("net_pins", np.int32, (E,)), ("sources", np.int32, (S,)), ("endpoints", np.int32, (EP,)),
            ("cell_fixed", np.uint8, (C,)), ("pos_explicit", np.uint8, (C,)), ("pin_dir", np.uint8, (P,))]


def save_bin(d: "Design", path: str) -> None:
    """Write ``d`` as a binary design file (layout above)."""
    counts = (d.n_cells, d.n_pins, d.n_nets, d.n_net_pins, int(d.sources.size), int(d.endpoints.size))
    flags = 1 if d.pin_names is not None else 0
    hdr = bytearray(BIN_HEADER)
    hdr[0:8] = BIN_MAGIC
    hdr[8:16] = np.array([1, flags], "<u4").tobytes()
    hdr[16:64] = np.array(counts, "<i8").tobytes()
    hdr[64:128] = np.array([d.clock_period, d.r_unit, d.c_unit, *d.core, d.default_cell_delay], "<f8").tobytes()
    with open(path, "wb") as f:
        f.write(hdr)
        for name, dt, shape in _bin_sections(counts):
            a = np.ascontiguousarray(getattr(d, name), dtype=np.dtype(dt).newbyteorder("<")).reshape(shape)
            b = a.tobytes()
            f.write(b)
            f.write(b"\0" * (-len(b) % 8))
        if flags & 1:
            blob = b"".join(n.encode() + b"\0" for n in d.pin_names)
            f.write(np.array([len(blob)], "<u8").tobytes())
            f.write(blob)


def load_bin(path: str) -> "Design":
    """Read a binary design file (layout above)."""
    buf = np.fromfile(path, dtype=np.uint8)
    if buf.size < BIN_HEADER or bytes(buf[:8]) != BIN_MAGIC:
        raise ValueError(f"parse error: {path}: not a binary design file")
    version, flags = np.frombuffer(buf[8:16].tobytes(), "<u4")
    if version != 1:
        raise ValueError(f"parse error: {path}: unsupported binary design version {version}")
    counts = tuple(int(x) for x in np.frombuffer(buf[16:64].tobytes(), "<i8"))
    if min(counts) < 0 or counts[2] < 0:
        raise ValueError(f"parse error: {path}: negative sizes")
    sc = np.frombuffer(buf[64:128].tobytes(), "<f8")
    off, kw = BIN_HEADER, {}
    for name, dt, shape in _bin_sections(counts):
        n = int(np.prod(shape)) * np.dtype(dt).itemsize
        if off + n > buf.size:
            raise ValueError(f"parse error: {path}: truncated ({name})")
        kw[name] = np.frombuffer(buf[off:off + n].tobytes(), np.dtype(dt).newbyteorder("<")).astype(dt).reshape(shape)
        off += n + (-n % 8)
    pin_names = None
    if flags & 1:
        nb = int(np.frombuffer(buf[off:off + 8].tobytes(), "<u8")[0])
        blob = bytes(buf[off + 8:off + 8 + nb])
        pin_names = [s.decode() for s in blob.split(b"\0")[:-1]]
        if len(pin_names) != counts[1]:
            raise ValueError(f"parse error: {path}: pin name count")
    return Design(clock_period=float(sc[0]), r_unit=float(sc[1]), c_unit=float(sc[2]), core=tuple(sc[3:7]),
                  default_cell_delay=float(sc[7]), pin_names=pin_names, **kw)
