"""ncu driver: one engine timing refresh (STA push sweep + extraction + ledger) of the 1M design inside
cudaProfilerStart/Stop, plus the GP iteration that follows it."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_11674_b200.engine import Session, generate  # noqa: E402

d = generate(seed=1, cells=int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, fail_frac=0.8, calibrate=True)
s = Session(d)
s.engine_init({"grid_nx": 1024, "grid_ny": 1024, "m": 15, "timing_start_iter": 0, "max_iters": 100, "seed": 1})
s.iterate(30)  # refreshes at 0, 15; the ledger is populated
torch.cuda.synchronize()
torch.cuda.profiler.start()
s.iterate(1)   # iteration 30: refresh + one GP iteration
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(s.engine_stats(), flush=True)
