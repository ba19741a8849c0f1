"""Device time per GP iteration (no timing refresh) of the captured iteration graph, 1M design."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_11674_b200.engine import Session, generate  # noqa: E402

d = generate(seed=1, cells=int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, fail_frac=0.8, calibrate=True)
s = Session(d)
s.engine_init({"grid_nx": 1024, "grid_ny": 1024, "m": 15, "timing_start_iter": 100000, "max_iters": 400, "seed": 1,
               "density_model": os.environ.get("DENSITY_MODEL", "overflow")})
s.iterate(20)
ms = min(s.iterate(50) for _ in range(3)) / 50
print(f"model={os.environ.get('DENSITY_MODEL', 'overflow')} iter_ms={ms:.4f}", flush=True)
