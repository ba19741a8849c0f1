"""Session-creation phase times on the bench's 1M design (TDPG_TRACE_CREATE=1 prints them)."""
import os
import sys
import time
import types

os.environ["TDPG_TRACE_CREATE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_11674_b200.engine import Session  # noqa: E402

args = types.SimpleNamespace(cells=int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, grid=1024, m=15,
                             warmup=20, steps=20, fail_frac=0.8)
d, _ = bench.make_design(args)
for _ in range(2):
    t0 = time.perf_counter()
    s = Session(d)
    print(f"session_create {1000 * (time.perf_counter() - t0):.1f} ms", flush=True)
    s.close()
