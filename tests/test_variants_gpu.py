"""The A/B switches of the hot path compute the same results bit for bit (each variant in its own process,
since the switches are read once): the density scatter's no-return limb adds against the carry-propagating
two-word form (same int64 grid, so the same value, overflow and cell gradient — spread, clumped and fully
stacked placements, on both sides of the 2-/3-limb threshold), and the 32-bit endpoint sort
with its run fix-up against the full 64-bit sort (same violated-endpoint order, so the same paths)."""
import hashlib
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r"""
import hashlib, sys
sys.path.insert(0, {root!r})
import numpy as np
from paper_2503_11674_b200.engine import Session, generate
d = generate(seed=7, cells={cells}, fail_frac=0.6, calibrate=False)
rng = np.random.default_rng(1)
x0, y0, x1, y1 = d.core
xy = d.positions.copy()
xy[:, 0] = x0 + rng.random(d.n_cells) * (x1 - x0 - d.cell_w)  # spread: windowed and fallback blocks
xy[:, 1] = y0 + rng.random(d.n_cells) * (y1 - y0 - d.cell_h)
xy[: d.n_cells // 3] = d.positions[: d.n_cells // 3]          # and a clumped third
s = Session(d)
h = hashlib.sha256()
for g in (16, 64, 256):
    v, o, dc = s.density(xy, nx=g, ny=g, td=0.6)
    h.update(np.float64([v, o]).tobytes()); h.update(dc.tobytes())
stack = np.tile([(x0 + x1) / 2, (y0 + y1) / 2], (d.n_cells, 1))  # every cell on one spot: full-block bins
v, o, dc = s.density(stack, nx=64, ny=64, td=0.6)
h.update(np.float64([v, o]).tobytes()); h.update(dc.tobytes())
r = s.extract(xy, n=0)
h.update(r["pins"].tobytes()); h.update(r["slack"].tobytes())
print(h.hexdigest())
"""


def _run(env_extra, cells):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", SNIPPET.format(root=ROOT, cells=cells)], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


@pytest.mark.parametrize("cells", [3000, 12000, 30000, 60000])
def test_switch_variants_bitwise(cells):
    base = _run({}, cells)
    assert _run({"TDPG_SCATTER_LIMBS": "0"}, cells) == base
    assert _run({"TDPG_EP_SORT64": "1"}, cells) == base
