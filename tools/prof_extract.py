"""ncu driver: one STA + top-n endpoint extraction (the bench's extraction sweep call) on the 1M design,
spread snapshot, 80% failing endpoints, inside cudaProfilerStart/Stop.  Usage: prof_extract.py [n]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_11674_b200.engine import Session, generate  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
d = generate(seed=1, cells=1_000_000, fail_frac=0.8, calibrate=False)
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
for _ in range(3):
    s.extract(None, n=n, run_sta=True)
torch.cuda.synchronize()
torch.cuda.profiler.start()
r = s.extract(None, n=n, run_sta=True)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(r["sta_ms"], r["extract_ms"], r["n_paths"], flush=True)
