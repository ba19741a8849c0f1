"""ncu driver: one STA of the 1M design inside cudaProfilerStart/Stop (per-level kernel durations)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_11674_b200.engine import Session, generate  # noqa: E402

d = generate(seed=1, cells=int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, fail_frac=0.8, calibrate=False)
s = Session(d)
s.sta()
s.sta()
torch.cuda.synchronize()
torch.cuda.profiler.start()
s.sta()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
