"""One process per GPU for the single-design partitioned mode and the replica mode.

torch.distributed is plumbing only: it carries the 128-byte NCCL unique id from rank 0 to the other
ranks and takes the max of per-rank device times.  The gradient all-reduce itself is issued by the
engine (ncclAllReduce captured inside its iteration graph), not by torch.
"""
from __future__ import annotations

import os

from . import engine


def rank_env():
    """(rank, world, local_rank) from the torchrun environment (1 process when unset)."""
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def broadcast_unique_id(rank: int, make_id=engine.comm_unique_id) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank returns the same 128 bytes."""
    import torch.distributed as dist
    box = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    uid = box[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad NCCL unique id from rank 0")
    return bytes(uid)


def init_partitioned(session: "engine.Session", rank: int, world: int) -> None:
    """Give `session` this rank's share of the nets and an NCCL communicator over all ranks."""
    if world > 1:
        uid = broadcast_unique_id(rank)
    else:  # (a one-rank communicator only when TDPG_COMM_WORLD1 asks for one: it needs a real id)
        uid = engine.comm_unique_id() if os.environ.get("TDPG_COMM_WORLD1") else bytes(128)
    session.comm_init(rank, world, uid)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device time of the timed region) over all ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def plan_covers(net_start, world: int):
    """The partition plan's block ranges tile the WA block list; returns (bounds, entries per rank)."""
    bounds, ent = engine.partition_plan(net_start, world)
    full = engine.partition_plan(net_start, 1)[0]
    assert bounds[0] == 0 and bounds[-1] == full[1] and all(bounds[i] <= bounds[i + 1] for i in range(world))
    return bounds, ent
