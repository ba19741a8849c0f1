"""ncu driver: the bench workload (bench.py make_design, 1M cells) up to its first timed iteration, then
ONE iteration holding a timing refresh inside cudaProfilerStart/Stop (run under ncu
--profile-from-start off; TDPG_NO_COND=1 makes the refresh graph's size-class bodies visible).
Usage: prof_refresh.py [warmup] [cells] [timing_start]  (timing_start defaults to warmup: the first refresh;
a warmup of timing_start + 15 k profiles a later one)"""
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_11674_b200.engine import Session  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cells = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
T0 = int(sys.argv[3]) if len(sys.argv) > 3 else W
args = types.SimpleNamespace(cells=cells, grid=1024 if cells >= 500000 else 512, m=15, warmup=T0, steps=20,
                             fail_frac=0.8)
d, _ = bench.make_design(args)
s = Session(d)
s.engine_init(bench.bench_config(args, W + 40))
s.iterate(W)
torch.cuda.synchronize()
torch.cuda.profiler.start()
ms = s.iterate(1)  # iteration W: refresh + GP iteration
torch.cuda.synchronize()
torch.cuda.profiler.stop()
st = s.engine_stats()
print(f"iteration with refresh: {ms:.3f} ms; paths {st['paths']} refresh_ms {st['refresh_ms']:.3f}", flush=True)
