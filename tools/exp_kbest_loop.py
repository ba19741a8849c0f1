"""The paper's rpt_timing_ept(n, k) ablation inside the device loop: the bench's 1M design, timing from the
first iteration, a refresh every 15, k = 1 versus k = 10 (both one captured refresh graph, host-sync-free),
and topn (host-driven list growth) for contrast: device ms per iteration and per refresh."""
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_11674_b200.engine import Session  # noqa: E402

args = types.SimpleNamespace(cells=int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, grid=1024, m=15, warmup=0,
                             steps=200, fail_frac=0.8)
d, _, _ = bench.load_or_make(args, bench.make_design)
for extra in ({"k": 1}, {"k": 10}, {"k": 10}, {"extraction": "topn", "k": 1}):
    cfg = dict(bench.bench_config(args, 200), timing_start_iter=0, **extra)
    s = Session(d)
    s.engine_init(cfg)
    ms = s.iterate(90)
    st = s.engine_stats()
    print(extra, f"{ms / 90:.4f} ms/iter, {st['refreshes']} refreshes at {st['refresh_ms'] / max(st['refreshes'], 1):.3f} ms,"
          f" paths {st['paths']}, ledger pairs {st['ledger_pairs']}", flush=True)
    s.close()
