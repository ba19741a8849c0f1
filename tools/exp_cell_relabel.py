"""Experiment: GP-iteration kernel times on the bench's 1M design with the cells relabelled (a pure
renaming of the input: pin_cell and the per-cell arrays permuted) — identity, random, and first touch in
net order (driver then sinks).  Tells how much of WA / density / cells depends on id locality."""
import copy
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2503_11674_b200.engine import Session  # noqa: E402


def relabel_cells(d, order):
    """order[new] = old."""
    inv = np.empty_like(order)
    inv[order] = np.arange(order.size)
    e = copy.copy(d)
    for k in ("cell_w", "cell_h", "cell_delay", "cell_fixed", "pos_explicit"):
        setattr(e, k, np.ascontiguousarray(getattr(d, k)[order]))
    e.positions = np.ascontiguousarray(d.positions[order])
    pc = d.pin_cell.copy()
    m = pc >= 0
    pc[m] = inv[pc[m]]
    e.pin_cell = pc.astype(np.int32)
    return e


def first_touch(d):
    seen = np.zeros(d.n_cells, bool)
    out = []
    cells = d.pin_cell[d.net_pins]
    for c in cells:
        if c >= 0 and not seen[c]:
            seen[c] = True
            out.append(c)
    out += list(np.nonzero(~seen)[0])
    return np.asarray(out, np.int64)


args = types.SimpleNamespace(cells=int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, grid=1024, m=15,
                             warmup=20, steps=20, fail_frac=0.8)
d, _ = bench.make_design(args)
orders = {"identity": np.arange(d.n_cells), "random": np.random.default_rng(0).permutation(d.n_cells),
          "first_touch": first_touch(d)}
for name, order in orders.items():
    e = relabel_cells(d, order)
    s = Session(e)
    s.engine_init(bench.bench_config(args, 400))
    s.iterate(40)
    ms = s.iterate(45) / 45
    prof = s.profile_iteration(5)
    print(name, f"{ms:.4f} ms/iter", {k: round(v * 1000, 1) for k, v in prof.items()}, flush=True)
    s.close()
