"""Device time per GP iteration along the bench's run (1M design, refresh every 15 iterations), in
blocks of 10 iterations: how the iteration cost moves as the cells spread from the jittered start."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_11674_b200.engine import Session, generate  # noqa: E402

d = generate(seed=1, cells=1_000_000, fail_frac=0.8, calibrate=True)
s = Session(d)
refresh = len(sys.argv) > 1 and sys.argv[1] == "refresh"
s.engine_init({"grid_nx": 1024, "grid_ny": 1024, "m": 15, "timing_start_iter": 0 if refresh else 100000,
               "max_iters": 400, "seed": 1})
out = []
for b in range(24):
    out.append(s.iterate(10) / 10)
print(" ".join(f"{m:.3f}" for m in out), flush=True)
