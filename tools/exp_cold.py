"""Cold end-to-end breakdown on the bench's 1M design: a fresh session + one run_placement call (tdpg_place)
with host buffers, twice in one process (the second excludes process-level first-use costs), with the
session-creation and engine_init phase traces on stderr."""
import os
import sys
import time
import types

os.environ["TDPG_TRACE_CREATE"] = "1"
os.environ["TDPG_TRACE_INIT"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_11674_b200.engine import Session  # noqa: E402

args = types.SimpleNamespace(cells=1_000_000, grid=1024, m=15, warmup=20, steps=200, fail_frac=0.8)
d, _, _ = bench.load_or_make(args, bench.make_design)
C = d.n_cells
hin = torch.empty(2 * C, dtype=torch.float64, pin_memory=True)
hout = torch.empty(2 * C, dtype=torch.float64, pin_memory=True)
hin.numpy()[:] = d.positions.reshape(-1)
cfg = dict(bench.bench_config(args, 200), timing_start_iter=0)
for r in range(2):
    t0 = time.perf_counter()
    s = Session(d)
    t1 = time.perf_counter()
    n, _ = s.place_host(cfg, hin.data_ptr(), hout.data_ptr())
    t2 = time.perf_counter()
    n2, _ = s.place_host(cfg, hin.data_ptr(), hout.data_ptr())
    t3 = time.perf_counter()
    print(f"cold {r}: create {1e3 * (t1 - t0):.1f} ms, first place {1e3 * (t2 - t1):.1f} ms ({n} iters), "
          f"second place {1e3 * (t3 - t2):.1f} ms", flush=True)
    s.close()
