"""N > 1 host logic on CPU (gloo, world_size 2): NCCL unique-id hand-off, the net partition plan every
rank derives independently, max-over-ranks timing.  The device path itself is covered on one GPU by
tests/test_partition_gpu.py (split-phase engine, reduction done by the test)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_11674_b200 import distributed as D
    from paper_2503_11674_b200.engine import generate
    d = generate(seed=1, cells=20000, calibrate=False)  # host-side generator: no GPU needed
    uid = D.broadcast_unique_id(rank)
    bounds, ent = D.plan_covers(d.net_start, world)
    t = D.max_over_ranks(1.5 + rank)
    out.put((rank, uid, bounds.tolist(), ent.tolist(), t, int(d.n_net_pins)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_handoff_plan_and_timing():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, u0, b0, e0, t0, E), (r1, u1, b1, e1, t1, _) = res
    assert u0 == u1 and len(u0) == 128          # every rank got rank 0's NCCL id
    assert b0 == b1 and e0 == e1                 # identical plans, derived independently
    assert sum(e0) == E                          # every net-pin entry owned by exactly one rank
    assert abs(e0[0] - e0[1]) <= 0.05 * E        # balanced by entries
    assert t0 == t1 == 2.5                       # max over ranks


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_plan_tiles_blocks(world):
    from paper_2503_11674_b200 import distributed as D
    from paper_2503_11674_b200.engine import generate
    d = generate(seed=2, cells=50000, calibrate=False)
    bounds, ent = D.plan_covers(d.net_start, world)
    assert int(np.sum(ent)) == int(d.n_net_pins)
    if world > 1:
        assert np.max(ent) <= 1.15 * d.n_net_pins / world
