"""ncu driver: one electrostatic density evaluation (scatter, bins, DCT Poisson solve, energy, gradient) on
the bench's 1M design at grid 1024^2 inside cudaProfilerStart/Stop (run under ncu --profile-from-start off)."""
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_11674_b200.engine import Session  # noqa: E402

args = types.SimpleNamespace(cells=1_000_000, grid=1024, m=15, warmup=20, steps=200, fail_frac=0.8)
d, _, _ = bench.load_or_make(args, bench.make_design)
s = Session(d)
s.set_density_model("electrostatic")
s.density(d.positions, nx=1024, ny=1024, td=0.6)
torch.cuda.synchronize()
torch.cuda.profiler.start()
s.density(d.positions, nx=1024, ny=1024, td=0.6)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
