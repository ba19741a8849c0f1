import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_11674_b200.engine import Session, generate
d = generate(seed=1, cells=1_000_000, fail_frac=0.8, calibrate=True)
s = Session(d)
s.engine_init({"grid_nx": 1024, "grid_ny": 1024, "m": 15, "timing_start_iter": 0, "max_iters": 300, "seed": 1})
for k in range(16):
    ms = s.iterate(15)
    st = s.engine_stats()
    print(f"chunk {k}: {ms:.2f} ms / 15 it; last refresh {st['last_refresh_ms']:.2f} ms; ledger {st['ledger_pairs']}", flush=True)
