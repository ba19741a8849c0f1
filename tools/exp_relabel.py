"""Experiment: STA device time on the 1M design with pins relabelled level-major (pin id order = level
order, Outputs before Inputs inside a level) versus the generator's order."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle.oracle import Oracle  # noqa: E402
from paper_2503_11674_b200.engine import Session, generate  # noqa: E402


def relabel(d, order):
    """Design with pin p renamed to inv[p] (order[new] = old)."""
    import copy
    inv = np.empty_like(order)
    inv[order] = np.arange(order.size)
    e = copy.copy(d)
    for k in ("pin_cell", "pin_dir", "pin_cap"):
        setattr(e, k, np.ascontiguousarray(getattr(d, k)[order]))
    for k in ("pin_term", "pin_off"):
        setattr(e, k, np.ascontiguousarray(getattr(d, k)[order]))
    e.net_pins = np.ascontiguousarray(inv[d.net_pins]).astype(np.int32)
    e.sources = np.ascontiguousarray(inv[d.sources]).astype(np.int32)
    e.endpoints = np.ascontiguousarray(inv[d.endpoints]).astype(np.int32)
    if getattr(d, "pin_names", None):
        e.pin_names = [d.pin_names[o] for o in order]
    return e


d = generate(seed=1, cells=int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, fail_frac=0.8, calibrate=False)
lvl = Oracle(d).graph()["level"]
order = np.lexsort((np.arange(d.n_pins), -d.pin_dir.astype(np.int64), lvl))
e = relabel(d, order)
for name, des in (("generator order", d), ("level-major", e)):
    s = Session(des)
    s.sta()
    best = min(s.extract(None, n=10000, run_sta=True)["sta_ms"] for _ in range(5))
    print(f"{name}: sta {best:.3f} ms", flush=True)
