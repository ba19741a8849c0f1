"""Electrostatic density (electro.cu).  Not in the reference, so no oracle: the
potential is checked against an independent 5-point Neumann stencil (L psi = rho - mean rho), the
gradient against central finite differences of the energy, and a placement run against the physics
(cells spread: overflow falls)."""
import numpy as np
import pytest

from fixtures import spread_positions
from paper_2503_11674_b200.engine import Session, generate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def design():
    return generate(seed=4, cells=2000, fail_frac=0.5, calibrate=False)


def _stencil(psi, bw, bh):
    q = np.pad(psi, 1, mode="edge")  # Neumann boundary: mirrored ghost cells
    return (2 * psi - q[:-2, 1:-1] - q[2:, 1:-1]) / bw ** 2 + (2 * psi - q[1:-1, :-2] - q[1:-1, 2:]) / bh ** 2


@pytest.mark.parametrize("nx,ny", [(32, 32), (64, 48), (20, 12), (7, 5), (1024, 1024), (256, 96), (128, 2048), (2048, 64), (64, 512), (4096, 32)])
def test_poisson_residual(design, nx, ny):
    s = Session(design)
    s.set_density_model("electrostatic")
    xy = spread_positions(design, 1)
    v, ov, _ = s.density(xy, nx=nx, ny=ny, td=0.6)
    rho, psi = s.density_fields(nx, ny)
    x0, y0, x1, y1 = design.core
    bw, bh = (x1 - x0) / nx, (y1 - y0) / ny
    res = _stencil(psi, bw, bh) - (rho - rho.mean())
    assert np.max(np.abs(res)) <= 1e-9 * np.max(np.abs(rho - rho.mean()))
    assert abs(psi.mean()) <= 1e-12 * np.max(np.abs(psi))
    assert v == pytest.approx(0.5 * np.sum(rho * psi), rel=1e-10) and v > 0.0
    # the overflow metric is the model-independent one
    s2 = Session(design)
    _, ov2, _ = s2.density(xy, nx=nx, ny=ny, td=0.6)
    assert ov == pytest.approx(ov2, rel=1e-12)


def test_energy_gradient_finite_differences(design):
    s = Session(design)
    s.set_density_model("electrostatic")
    xy = spread_positions(design, 2)
    nx = ny = 32
    _, _, g = s.density(xy, nx=nx, ny=ny, td=0.6)
    rng = np.random.default_rng(0)
    h = 1e-3 * (design.core[2] - design.core[0]) / nx
    movable = np.flatnonzero(design.cell_fixed == 0)
    for c in rng.choice(movable, 12, replace=False):
        for ax in (0, 1):
            xp, xm = xy.copy(), xy.copy()
            xp[c, ax] += h
            xm[c, ax] -= h
            fd = (s.density(xp, nx=nx, ny=ny, td=0.6)[0] - s.density(xm, nx=nx, ny=ny, td=0.6)[0]) / (2 * h)
            assert abs(fd - g[c, ax]) <= 1e-5 * np.max(np.abs(g)), (c, ax, fd, g[c, ax])


def test_electrostatic_placement_spreads(design):
    cfg = {"max_iters": 150, "timing_start_iter": 100000, "grid_nx": 32, "grid_ny": 32, "seed": 4,
           "density_model": "electrostatic"}
    out = Session(design).place(cfg)
    tr = out["trace"]
    assert len(tr) == 150 and all(np.isfinite(r.density_term) for r in tr)
    assert tr[-1].overflow < 0.5 * tr[0].overflow
