"""Row-by-row divergence of the GPU placement trajectory from the oracle's."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.oracle import Oracle, RefOracle
from paper_2503_11674_b200.engine import Session, generate

d = RefOracle.generate(seed=2, cells=2000, fail_frac=0.4) if RefOracle.available() else generate(seed=2, cells=2000, fail_frac=0.4, calibrate=False)
d.clock_period = 1.0
for cfg in [{"max_iters": 300, "timing_start_iter": 300, "beta": 0.0, "seed": 2},
            {"max_iters": 300, "timing_start_iter": 300, "beta": 0.0, "seed": 2, "grid_nx": 64, "grid_ny": 64}]:
    ps, po = Session(d).place(cfg), Oracle(d).place(cfg)
    print("cfg", cfg)
    for i in [0, 1, 2, 3, 5, 10, 20, 40, 80, 120, 160, 200, 250, 299]:
        if i < len(po["trace"]):
            a, b = ps["trace"][i], po["trace"][i]
            print(f"  it {i:3d} hpwl rel {abs(a.hpwl-b.hpwl)/b.hpwl:.3e} ovf rel {abs(a.overflow-b.overflow)/max(b.overflow,1e-30):.3e} "
                  f"lam rel {abs(a.lambda_-b.lambda_)/b.lambda_:.3e} dens rel {abs(a.density_term-b.density_term)/max(b.density_term,1e-30):.3e}")
    pos_err = np.max(np.abs(ps["positions"] - po["positions"]))
    print("  final pos max abs diff", pos_err, "tns", ps["tns"], po["tns"])
