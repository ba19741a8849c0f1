"""The partitioned single-design mode on one GPU: G sessions, one per rank, each
owning a net range and a slice of the cells' spatial order; the test performs both all-reduces (the
int64 density grid, then the gradient buffer: element-wise sums, the operations NCCL performs in the
multi-GPU graph) between the split phases.  Checks: the summed grid is bitwise the single-session grid,
ranks stay bitwise identical (replicated bins / Adam / timing refresh), and the trajectory equals the
single-session engine's to rounding (only the fold's summation order differs)."""
import numpy as np
import pytest

from paper_2503_11674_b200.engine import Session, generate, red_size

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def design():
    d = generate(seed=3, cells=3000, fail_frac=0.5, calibrate=True)
    d.clock_period *= 0.6  # make timing rounds engage early
    return d


def _run_split(d, cfg, world, iters):
    ss = []
    for r in range(world):
        s = Session(d)
        s.set_partition(r, world)
        s.engine_init(cfg)
        ss.append(s)
    n = red_size(ss[0])
    B = cfg["grid_nx"] * cfg["grid_ny"]
    bufs = [np.zeros(n) for _ in ss]
    accs = [np.zeros(B, np.int64) for _ in ss]
    for _ in range(iters):
        for s, a in zip(ss, accs):
            assert s.part_density_into(a) == B
        acc = np.sum(accs, axis=0)  # (int64: exact)
        for s, b in zip(ss, bufs):
            assert s.part_step_a_into(acc, b) == n
        total = bufs[0].copy()
        for b in bufs[1:]:
            total += b
        for s in ss:
            s.part_step_b(total)
    return ss



@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("extra", [{}, {"net_weighting": True, "pp_loss": "linear"}, {"k": 2}])
def test_partitioned_matches_single(design, world, extra):
    cfg = dict({"max_iters": 40, "timing_start_iter": 10, "m": 5, "grid_nx": 32, "grid_ny": 32, "seed": 3}, **extra)
    iters = 30
    ref = Session(design)
    ref.engine_init(cfg)
    ref.iterate(iters)
    xr = ref.positions()
    ss = _run_split(design, cfg, world, iters)
    xs = [s.positions() for s in ss]
    for x in xs[1:]:
        assert np.array_equal(x, xs[0])  # replicated optimizer: ranks never drift apart
    span = max(design.core[2] - design.core[0], design.core[3] - design.core[1])
    assert np.max(np.abs(xs[0] - xr)) <= 1e-7 * span
    st = ss[0].engine_stats()
    assert st["refreshes"] == ref.engine_stats()["refreshes"] > 0
    assert st["ledger_pairs"] == ref.engine_stats()["ledger_pairs"] > 0


def test_partitioned_requires_communicator(design):
    s = Session(design)
    s.set_partition(0, 2)
    s.engine_init({"max_iters": 5, "grid_nx": 16, "grid_ny": 16})
    with pytest.raises(Exception, match="communicator"):
        s.iterate(1)
