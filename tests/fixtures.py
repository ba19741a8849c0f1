"""Test designs, restating the reference's fixtures (proj/tests/fixtures.hpp).

T1 (:91-112), T2 (:119-147), diamond (:151-173), trunk16 (:182-220),
random_design (:268-347) — same ids, geometry and RNG stream (mt19937_64 +
include/tdp/rng.hpp helpers), so known answers from the reference tests apply.
"""
from __future__ import annotations

import numpy as np

from paper_2503_11674_b200.design import Design

_MASK = (1 << 64) - 1


class MT64:
    """std::mt19937_64."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & _MASK
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _MASK
        self.idx = 312

    def __call__(self):
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000 & _MASK
        y ^= (y << 37) & 0xFFF7EEE000000000 & _MASK
        y ^= y >> 43
        return y & _MASK

    def unit(self):
        return float(self() >> 11) * 2.0 ** -53

    def uniform(self, lo, hi):
        return lo + (hi - lo) * self.unit()

    def randint(self, lo, hi):
        return lo + self() % (hi - lo + 1)


class Builder:
    """DesignBuilder (fixtures.hpp:18-84)."""

    def __init__(self, core, clock, r_unit, c_unit):
        self.core, self.clock, self.r, self.c = core, clock, r_unit, c_unit
        self.cells, self.pins, self.nets, self.src, self.eps = [], [], [], [], []

    def cell(self, name, w, h, delay, pos, fixed=False):
        self.cells.append((name, w, h, delay, pos, fixed))
        return len(self.cells) - 1

    def pin(self, name, cell, out, cap=0.0, off=(0.0, 0.0)):
        self.pins.append((name, cell, (0.0, 0.0), off, out, cap))
        return len(self.pins) - 1

    def terminal(self, name, pos, out, cap=0.0):
        self.pins.append((name, -1, pos, (0.0, 0.0), out, cap))
        return len(self.pins) - 1

    def net(self, name, driver, sinks):
        self.nets.append((name, driver, list(sinks)))
        return len(self.nets) - 1

    def finish(self) -> Design:
        ns, np_ = [0], []
        for _, d, s in self.nets:
            np_ += [d] + s
            ns.append(len(np_))
        cells = self.cells
        return Design(
            cell_w=[c[1] for c in cells], cell_h=[c[2] for c in cells], cell_delay=[c[3] for c in cells],
            cell_fixed=[1 if c[5] else 0 for c in cells], pin_cell=[p[1] for p in self.pins],
            pin_term=np.array([p[2] for p in self.pins], dtype=np.float64).reshape(-1, 2),
            pin_off=np.array([p[3] for p in self.pins], dtype=np.float64).reshape(-1, 2),
            pin_dir=[1 if p[4] else 0 for p in self.pins], pin_cap=[p[5] for p in self.pins], net_start=ns,
            net_pins=np_, sources=self.src, endpoints=self.eps, clock_period=self.clock, r_unit=self.r,
            c_unit=self.c, core=self.core, positions=np.array([c[4] for c in cells], dtype=np.float64).reshape(-1, 2),
            pos_explicit=[1] * len(cells), cell_names=[c[0] for c in cells], pin_names=[p[0] for p in self.pins],
            net_names=[n[0] for n in self.nets])


IN, OUT = False, True


def make_t1():
    b = Builder((0, 0, 10, 10), 10.0, 1.0, 1.0)
    a = b.cell("A", 1, 1, 1.0, (0, 0))
    bb = b.cell("B", 1, 1, 1.0, (3, 0))
    c = b.cell("C", 1, 1, 1.0, (3, 4))
    pi = b.terminal("PI", (0, 0), OUT)
    a_in, a_out = b.pin("A.in", a, IN), b.pin("A.out", a, OUT)
    b_in, b_out = b.pin("B.in", bb, IN), b.pin("B.out", bb, OUT)
    c_in, c_out = b.pin("C.in", c, IN), b.pin("C.out", c, OUT)
    po = b.terminal("PO", (3, 4), IN)
    b.net("n0", pi, [a_in])
    b.net("n1", a_out, [b_in])
    b.net("n2", b_out, [c_in])
    b.net("n3", c_out, [po])
    b.src.append(pi)
    b.eps.append(po)
    return b.finish()


def make_t2():
    b = Builder((0, 0, 10, 10), 10.0, 1.0, 1.0)
    x = b.cell("X", 1, 1, 7.0, (0, 0))
    y = b.cell("Y", 1, 1, 6.0, (0, 0))
    z = b.cell("Z", 1, 1, 13.0, (0, 0))
    m = b.cell("M", 1, 1, 8.0, (0, 0))
    s = b.terminal("S", (0, 0), OUT)
    x_in, x_out = b.pin("X.in", x, IN), b.pin("X.out", x, OUT)
    y_in, y_out = b.pin("Y.in", y, IN), b.pin("Y.out", y, OUT)
    z_in, z_out = b.pin("Z.in", z, IN), b.pin("Z.out", z, OUT)
    m_a, m_b, m_out = b.pin("M.a", m, IN), b.pin("M.b", m, IN), b.pin("M.out", m, OUT)
    ep1, ep2 = b.terminal("EP1", (0, 0), IN), b.terminal("EP2", (0, 0), IN)
    b.net("nS", s, [x_in, y_in, z_in])
    b.net("nX", x_out, [m_a])
    b.net("nY", y_out, [m_b])
    b.net("nM", m_out, [ep1])
    b.net("nZ", z_out, [ep2])
    b.src.append(s)
    b.eps += [ep1, ep2]
    return b.finish()


def make_diamond(delay_a=7.0, delay_b=5.0):
    b = Builder((0, 0, 10, 10), 10.0, 1.0, 1.0)
    a = b.cell("A", 1, 1, delay_a, (0, 0))
    bb = b.cell("B", 1, 1, delay_b, (0, 0))
    m = b.cell("M", 1, 1, 1.0, (0, 0))
    s = b.terminal("S", (0, 0), OUT)
    a_in, a_out = b.pin("A.in", a, IN), b.pin("A.out", a, OUT)
    b_in, b_out = b.pin("B.in", bb, IN), b.pin("B.out", bb, OUT)
    m_a, m_b, m_out = b.pin("M.a", m, IN), b.pin("M.b", m, IN), b.pin("M.out", m, OUT)
    ep = b.terminal("EP", (0, 0), IN)
    b.net("nS", s, [a_in, b_in])
    b.net("nA", a_out, [m_a])
    b.net("nB", b_out, [m_b])
    b.net("nM", m_out, [ep])
    b.src.append(s)
    b.eps.append(ep)
    return b.finish()


def make_trunk16():
    b = Builder((0, 0, 10, 10), 30.0, 1.0, 1.0)
    s = b.terminal("S", (0, 0), OUT)
    b.src.append(s)
    prev = s
    for k in range(1, 5):
        sk = str(k)
        a = b.cell("A" + sk, 1, 1, 5.0 + 0.001 * (1 << (k - 1)), (0, 0))
        bb = b.cell("B" + sk, 1, 1, 5.0, (0, 0))
        m = b.cell("M" + sk, 1, 1, 1.0, (0, 0))
        a_in, a_out = b.pin("A" + sk + ".in", a, IN), b.pin("A" + sk + ".out", a, OUT)
        b_in, b_out = b.pin("B" + sk + ".in", bb, IN), b.pin("B" + sk + ".out", bb, OUT)
        m_a, m_b = b.pin("M" + sk + ".a", m, IN), b.pin("M" + sk + ".b", m, IN)
        m_out = b.pin("M" + sk + ".out", m, OUT)
        b.net("in" + sk, prev, [a_in, b_in])
        b.net("a" + sk, a_out, [m_a])
        b.net("b" + sk, b_out, [m_b])
        prev = m_out
    ins = []
    for j in range(1, 17):
        sj = str(j)
        e = b.cell("E" + sj, 1, 1, 10.0 + j, (0, 0))
        e_in, e_out = b.pin("E" + sj + ".in", e, IN), b.pin("E" + sj + ".out", e, OUT)
        t = b.terminal("T" + sj, (0, 0), IN)
        ins.append(e_in)
        b.net("e" + sj, e_out, [t])
        b.eps.append(t)
    b.net("fan", prev, ins)
    return b.finish()


def random_design(seed, max_cells=12):
    """fixtures.hpp:268-347, same mt19937_64 stream."""
    rng = MT64(seed)
    core = (0.0, 0.0, 20.0, 20.0)
    # DesignBuilder(core, clock, r, c): g++ evaluates these arguments right to left
    c_u = rng.uniform(0.1, 1.0)
    r_u = rng.uniform(0.1, 1.0)
    clock = rng.uniform(5.0, 50.0)
    b = Builder(core, clock, r_u, c_u)
    n_pi = rng.randint(1, 2)
    drivers = []
    for i in range(n_pi):
        pos = (core[0], rng.uniform(core[1], core[3]))
        p = b.terminal(f"pi{i}", pos, OUT)
        b.src.append(p)
        drivers.append(p)
    n_layers = rng.randint(2, 4)
    made = 0
    with_register = rng.unit() < 0.5
    register_slot = rng.randint(1, max(1, max_cells // 2)) if with_register else -1
    conns = []
    layer = 0
    while layer < n_layers and made < max_cells:
        width = rng.randint(1, 3)
        outs = []
        i = 0
        while i < width and made < max_cells:
            name = f"c{made}"
            w = rng.uniform(1.0, 2.0)
            h = rng.uniform(1.0, 2.0)
            px = rng.uniform(core[0], core[2] - w)
            py = rng.uniform(core[1], core[3] - h)
            cell = b.cell(name, w, h, rng.uniform(0.1, 2.0), (px, py))
            is_reg = made == register_slot and layer > 0
            n_in = 1 if is_reg else rng.randint(1, 2)
            first_in = -1
            for j in range(n_in):
                ox = rng.uniform(0.0, w)  # braced offset argument is evaluated before the cap (g++ order)
                oy = rng.uniform(0.0, h)
                cap = rng.uniform(0.0, 2.0)
                p = b.pin(f"{name}.i{j}", cell, IN, cap, (ox, oy))
                if j == 0:
                    first_in = p
                conns.append((p, drivers[rng.randint(0, len(drivers) - 1)]))
            ox = rng.uniform(0.0, w)
            oy = rng.uniform(0.0, h)
            out = b.pin(f"{name}.o", cell, OUT, 0.0, (ox, oy))
            if is_reg:
                b.eps.append(first_in)
                b.src.append(out)
            outs.append(out)
            i += 1
            made += 1
        drivers += outs
        layer += 1
    n_po = rng.randint(1, 2)
    for i in range(n_po):
        pos = (core[2], rng.uniform(core[1], core[3]))
        p = b.terminal(f"po{i}", pos, IN, rng.uniform(0.0, 2.0))
        b.eps.append(p)
        conns.append((p, drivers[rng.randint(0, len(drivers) - 1)]))
    for drv in drivers:
        sinks = [s for s, d in conns if d == drv]
        if sinks:
            b.net(f"n{len(b.nets)}", drv, sinks)
    d = b.finish()
    d.validate()
    return d


def spread_positions(design, seed=1):
    """Positions uniform over the core (a 'spread' snapshot), fixed cells untouched."""
    rng = np.random.default_rng(seed)
    x0, y0, x1, y1 = design.core
    pos = design.positions.copy()
    mov = design.cell_fixed == 0
    pos[mov, 0] = x0 + rng.random(mov.sum()) * (x1 - x0 - design.cell_w[mov])
    pos[mov, 1] = y0 + rng.random(mov.sum()) * (y1 - y0 - design.cell_h[mov])
    return pos
