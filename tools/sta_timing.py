"""STA + top-k extraction device time on a 1M design (spread snapshot, 80% failing endpoints)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2503_11674_b200.engine import Session, generate  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
d = generate(seed=1, cells=cells, fail_frac=0.8, calibrate=False)
rng = np.random.default_rng(1)
xy = d.positions.copy()
x0, y0, x1, y1 = d.core
xy[:, 0] = x0 + rng.random(d.n_cells) * (x1 - x0 - d.cell_w)
xy[:, 1] = y0 + rng.random(d.n_cells) * (y1 - y0 - d.cell_h)
s = Session(d)
t = s.sta(xy)
d.clock_period = float(np.quantile(t["arr"][d.endpoints], 0.2))
s = Session(d)
s.set_positions(xy)
for n in (1000, 10000, 100000):
    best = min((s.extract(None, n=n, run_sta=True) for _ in range(5)), key=lambda r: r["sta_ms"] + r["extract_ms"])
    print(f"env {os.environ.get('TDPG_STA_PERSIST', '1')}/{os.environ.get('TDPG_STA_BLOCKS_PER_SM', '2')} n={n}: "
          f"sta {best['sta_ms']:.3f} ms extract {best['extract_ms']:.3f} ms paths {best['n_paths']}", flush=True)
r = s.extract(None, n=10000, k=4, run_sta=False)
print(f"k=4 n=10000: extract {r['extract_ms']:.3f} ms paths {r['n_paths']}", flush=True)
