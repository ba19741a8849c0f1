"""The partitioned single-design engine driven by two processes, both on cuda:0, with the
two reductions of every iteration done over torch.distributed (gloo): the int64 density grid (each rank
rasterises its slice of the cells) and the partial cell gradient + objective partials.  This is the
multi-GPU data path with NCCL replaced by gloo: ranks must end bitwise identical and on the single-GPU
engine's trajectory to rounding."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CFG = {"max_iters": 40, "timing_start_iter": 10, "m": 5, "grid_nx": 32, "grid_ny": 32, "seed": 3}
ITERS = 30


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _design():
    from paper_2503_11674_b200.engine import generate
    d = generate(seed=3, cells=3000, fail_frac=0.5, calibrate=True)
    d.clock_period *= 0.6
    return d


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_11674_b200.engine import Session, red_size
    d = _design()
    s = Session(d)
    s.set_partition(rank, world)
    s.engine_init(CFG)
    B = CFG["grid_nx"] * CFG["grid_ny"]
    n = red_size(s)
    acc = np.zeros(B, np.int64)
    red = np.zeros(n)
    for _ in range(ITERS):
        s.part_density_into(acc)
        t = torch.from_numpy(acc)
        dist.all_reduce(t)  # int64 sum
        s.part_step_a_into(t.numpy(), red)
        t = torch.from_numpy(red)
        dist.all_reduce(t)
        s.part_step_b(t.numpy())
    st = s.engine_stats()
    q.put((rank, s.positions(), st["refreshes"], st["ledger_pairs"]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_partitioned_engine_over_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from paper_2503_11674_b200.engine import Session
    d = _design()
    ref = Session(d)
    ref.engine_init(CFG)
    ref.iterate(ITERS)
    xr = ref.positions()
    (_, x0, rf0, lp0), (_, x1, rf1, lp1) = res
    assert np.array_equal(x0, x1)  # replicated optimizer: the ranks never drift apart
    span = max(d.core[2] - d.core[0], d.core[3] - d.core[1])
    assert np.max(np.abs(x0 - xr)) <= 1e-7 * span
    st = ref.engine_stats()
    assert rf0 == rf1 == st["refreshes"] > 0
    assert lp0 == lp1 == st["ledger_pairs"] > 0
