import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_11674_b200.engine import Session, generate
d = generate(seed=1, cells=1_000_000, fail_frac=0.8, calibrate=True)
for se in ["1000000", "4", "2", "1"]:
    os.environ["TDPG_SORT_EVERY"] = se
    s = Session(d)
    cfg = {"grid_nx": 1024, "grid_ny": 1024, "m": 15, "timing_start_iter": 0, "max_iters": 400, "seed": 1}
    s.engine_init(cfg)
    s.iterate(20)
    ms = s.iterate(100)
    t0 = time.perf_counter(); ms2 = s.iterate(14); wall = time.perf_counter() - t0   # no refresh inside? (120..133)
    prof = s.profile_iteration(6)
    print(f"sort_every={se}: {ms/100:.3f} ms/iter (100 incl refresh); 14 iters {ms2/14:.3f} ms/iter wall {wall*1000/14:.3f}; prof {prof}", flush=True)
    s.close()
