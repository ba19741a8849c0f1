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


def test_nccl_graph_path_one_rank(design, monkeypatch):
    """The multi-GPU engine's own data path — NCCL all-reduces of the int64 density grid and the gradient
    buffer captured inside the iteration graph — on one GPU with a one-rank communicator (TDPG_COMM_WORLD1):
    the all-reduces are identities, so the run must reproduce the single-GPU engine (same fold order, same
    density gradient addition) row for row."""
    from paper_2503_11674_b200.engine import comm_unique_id
    monkeypatch.setenv("TDPG_COMM_WORLD1", "1")
    cfg = {"max_iters": 40, "timing_start_iter": 10, "m": 5, "grid_nx": 32, "grid_ny": 32, "seed": 3}
    ref = Session(design).place(cfg)
    s = Session(design)
    s.comm_init(0, 1, comm_unique_id())
    got = s.place(cfg)
    assert len(got["trace"]) == len(ref["trace"]) == 40
    assert any(r.has_timing and r.wns < 0 for r in ref["trace"])
    for rg, rr in zip(got["trace"], ref["trace"]):
        assert abs(rg.hpwl - rr.hpwl) <= 1e-9 * rr.hpwl, (rg.iter, rg.hpwl, rr.hpwl)
        assert abs(rg.tns - rr.tns) <= 1e-9 * max(1.0, abs(rr.tns)), (rg.iter, rg.tns, rr.tns)
    assert np.allclose(got["positions"], ref["positions"], rtol=0, atol=1e-9 * (design.core[2] - design.core[0]))
    s.comm_bench(5)  # (the two collectives alone, on the communicator)
