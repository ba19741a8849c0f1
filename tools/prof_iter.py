"""Small driver for ncu: a 1M design, engine warmed up for W iterations (default 17, two timing
refreshes), then a few plain GP iterations inside cudaProfilerStart/Stop (run ncu with
--profile-from-start off to capture only those)."""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_11674_b200.engine import Session, generate

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 17
n = int(sys.argv[3]) if len(sys.argv) > 3 else 5
d = generate(seed=1, cells=cells, fail_frac=0.8, calibrate=True)
s = Session(d)
grid = int(sys.argv[4]) if len(sys.argv) > 4 else 1024
s.engine_init({"grid_nx": grid, "grid_ny": grid, "m": 15, "timing_start_iter": 0, "max_iters": warm + 40, "seed": 1})
s.iterate(warm)
import torch  # noqa: E402  (cudaProfilerStart/Stop on the primary context the engine uses)
torch.cuda.synchronize()
print("profile window start", flush=True)
torch.cuda.profiler.start()
s.iterate(n)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(s.engine_stats(), flush=True)
