"""Fixed cost of one warm tdpg_place call on the bench's 1M design: wall time of the call against its
device loop, with the engine-init / place phase times (TDPG_TRACE_INIT=1 on stderr)."""
import os
import sys
import time
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_11674_b200.engine import Session  # noqa: E402

args = types.SimpleNamespace(cells=1_000_000, grid=1024, m=15, warmup=20, steps=200, fail_frac=0.8)
d, _ = bench.make_design(args)
s = Session(d)
C = d.n_cells
hin = torch.empty(2 * C, dtype=torch.float64, pin_memory=True)
hout = torch.empty(2 * C, dtype=torch.float64, pin_memory=True)
hin.numpy()[:] = d.positions.reshape(-1)
cfg = dict(bench.bench_config(args, 200), timing_start_iter=0)
s.place_host(cfg, hin.data_ptr(), hout.data_ptr())
for k in range(3):
    if k == 2:
        os.environ["TDPG_TRACE_INIT"] = "1"
    t0 = time.perf_counter()
    rows, _ = s.place_host(cfg, hin.data_ptr(), hout.data_ptr())
    dt = time.perf_counter() - t0
    print(f"call {k}: {rows} rows in {1000 * dt:.2f} ms -> {rows / dt:.0f} iters/s", flush=True)
s.engine_init(cfg, d.positions)
ms = s.iterate(200)
print(f"device loop alone: {ms:.2f} ms -> {200 / ms * 1000:.0f} iters/s", flush=True)
