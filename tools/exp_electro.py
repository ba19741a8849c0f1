"""GP iteration time on the bench's 1M design with the bin-overflow density (the reference's) and with
the electrostatic density (hand-written DCT Poisson solve, electro.cu) at grid 1024^2: the difference is
the cost of the solve + energy inside the iteration graph."""
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_11674_b200.engine import Session  # noqa: E402

args = types.SimpleNamespace(cells=1_000_000, grid=1024, m=15, warmup=20, steps=200, fail_frac=0.8)
d, _, _ = bench.load_or_make(args, bench.make_design)
res = {}
for model in ("overflow", "electrostatic", "overflow", "electrostatic"):
    cfg = dict(bench.bench_config(args, 400), timing_start_iter=100000, density_model=model)
    s = Session(d)
    s.engine_init(cfg)
    s.iterate(20)
    ms = s.iterate(100) / 100
    res[model] = min(res.get(model, 1e9), ms)
    s.close()
print({k: round(v, 4) for k, v in res.items()}, "electrostatic extra per iteration (us):",
      round(1000 * (res["electrostatic"] - res["overflow"]), 1), flush=True)
