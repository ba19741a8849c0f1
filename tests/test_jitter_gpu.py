"""The run's starting positions (placer.cpp:375-382): the device draws the std::mt19937_64 stream itself
(place.cu k_mt19937_64) and applies the jitter + core clamp per cell.  Bit-exact against the oracle's
sequential restatement, across many engine regenerations (312 draws each), with explicit and fixed
cells skipped, the clamp engaged, and 64-bit seeds."""
import numpy as np
import pytest

from fixtures import random_design
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu

from paper_2503_11674_b200.engine import Session, generate  # noqa: E402


def _start(d, cfg):
    s = Session(d)
    s.engine_init(cfg)
    return s.positions()


@pytest.mark.parametrize("seed", [1, 2, 5, 11])
def test_jitter_small_designs(seed):
    d = random_design(seed)
    cfg = {"seed": seed * 7919, "init_jitter_frac": 0.05, "grid_nx": 8, "grid_ny": 8, "max_iters": 3}
    assert np.array_equal(_start(d, cfg), Oracle(d).jitter(cfg))


@pytest.mark.parametrize("seed,frac", [(1, 0.02), (2**63 + 12345, 0.3), (0, 1.5)])
def test_jitter_generated_with_explicit_cells(seed, frac):
    d = generate(seed=3, cells=20000, fail_frac=0.5)
    rng = np.random.default_rng(seed % 1000)
    d.pos_explicit[:] = (rng.random(d.n_cells) < 0.2).astype(np.uint8)
    cfg = {"seed": seed, "init_jitter_frac": frac, "grid_nx": 32, "grid_ny": 32, "max_iters": 3}
    got, want = _start(d, cfg), Oracle(d).jitter(cfg)
    assert np.array_equal(got, want)
    moved = np.any(got != d.positions, axis=1)
    assert not np.any(moved & (d.pos_explicit != 0))
    assert moved.sum() > 0.5 * d.n_cells  # (a large frac clamps many cells onto the core boundary)


def test_jitter_zero_frac_and_all_explicit():
    d = generate(seed=4, cells=3000, fail_frac=0.5)
    cfg = {"seed": 9, "init_jitter_frac": 0.0, "grid_nx": 16, "grid_ny": 16, "max_iters": 3}
    assert np.array_equal(_start(d, cfg), Oracle(d).jitter(cfg))
    d.pos_explicit[:] = 1
    cfg["init_jitter_frac"] = 0.1
    assert np.array_equal(_start(d, cfg), d.positions)


def test_jitter_stream_reused_across_runs_of_a_session():
    """The session keeps the raw mt19937_64 stream per seed: later runs with the same seed (other
    explicit cells), then another seed, still start bitwise where the oracle does."""
    d = generate(seed=6, cells=8000, fail_frac=0.5)
    s = Session(d)
    cfg = {"seed": 77, "init_jitter_frac": 0.05, "grid_nx": 16, "grid_ny": 16, "max_iters": 2}
    for frac_explicit, seed in ((0.0, 77), (0.3, 77), (0.1, 77), (0.0, 78), (0.2, 77)):
        d.pos_explicit[:] = (np.random.default_rng(seed).random(d.n_cells) < frac_explicit).astype(np.uint8)
        cfg["seed"] = seed
        s.engine_init(cfg, xy=d.positions)
        assert np.array_equal(s.positions(), Oracle(d).jitter(cfg)), (frac_explicit, seed)
