import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2503_11674_b200.engine import Session, generate
d = generate(seed=1, cells=1_000_000, fail_frac=0.8, calibrate=True)
s = Session(d)
C = d.n_cells
hin = torch.empty(2 * C, dtype=torch.float64, pin_memory=True); hout = torch.empty_like(hin).pin_memory()
hin.numpy()[:] = d.positions.reshape(-1)
cfg = {"grid_nx": 1024, "grid_ny": 1024, "m": 15, "timing_start_iter": 0, "max_iters": 200, "seed": 1}
for r in range(3):
    t0 = time.perf_counter(); n, _ = s.place_host(cfg, hin.data_ptr(), hout.data_ptr()); t1 = time.perf_counter()
    print(f"run {r}: {n} iters in {t1-t0:.4f} s -> {n/(t1-t0):.1f} it/s", flush=True)
t0 = time.perf_counter(); s.engine_init(cfg); torch.cuda.synchronize(); print("engine_init", time.perf_counter()-t0)
import ctypes as C
t0 = time.perf_counter(); s.engine_init(cfg); torch.cuda.synchronize(); t1 = time.perf_counter()
s.iterate(200); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"engine_init {t1-t0:.4f} s, iterate(200) {t2-t1:.4f} s", flush=True)
t0 = time.perf_counter(); s.sta(); torch.cuda.synchronize(); print(f"final sta {time.perf_counter()-t0:.4f} s")
