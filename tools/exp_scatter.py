"""Density kernel times along the bench's run (1M design, refresh every 15): per-kernel device time of a
few iterations at several points of the run, from the clumped jittered start to spread placements.
Run once per scatter variant (TDPG_SCATTER=0/1)."""
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_11674_b200.engine import Session  # noqa: E402

args = types.SimpleNamespace(cells=int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, grid=1024, m=15,
                             warmup=20, steps=20, fail_frac=0.8)
d, _ = bench.make_design(args)
s = Session(d)
s.engine_init(bench.bench_config(args, 3000))
done = 0
for stop in (20, 60, 120, 220, 400, 700, 1000, 1500):
    s.iterate(stop - done)
    done = stop
    ms = s.iterate(10) / 10
    done += 10
    prof = s.profile_iteration(4)
    done += 4
    print(f"iter {stop:5d} {ms:.4f} ms/iter", {k: round(v * 1000, 1) for k, v in prof.items()}, flush=True)
