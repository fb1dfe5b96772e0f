"""Process-group plumbing for one process per GPU (bench.py and callers).

The engine shards observations by contiguous index ranges (comm.cu shard_rows); the NCCL
communicator is created from a unique id that rank 0 broadcasts over an existing
torch.distributed group.  Timings are reported as the max over ranks.  These helpers hold no
device state, so the CPU tests drive them with the gloo backend.
"""
from __future__ import annotations

import os


def env_ranks():
    """(world, rank, local_rank) from the torchrun environment (1, 0, 0 when absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n: int, rank: int, world: int):
    """Rows [lo, hi) owned by `rank` -- the same split as the engine's shard_rows (comm.cu)."""
    return n * rank // world, n * (rank + 1) // world


def broadcast_object(obj, src: int = 0):
    """Broadcast a picklable object from `src` over the default process group."""
    import torch.distributed as tdist
    box = [obj]
    tdist.broadcast_object_list(box, src=src)
    return box[0]


def max_over_ranks(value: float) -> float:
    """Max of a per-rank scalar (device-timed step times are reported as the slowest rank)."""
    import torch
    import torch.distributed as tdist
    if not (tdist.is_available() and tdist.is_initialized()) or tdist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t[0])


def sum_over_ranks(value: float) -> float:
    import torch
    import torch.distributed as tdist
    if not (tdist.is_available() and tdist.is_initialized()) or tdist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64)
    tdist.all_reduce(t, op=tdist.ReduceOp.SUM)
    return float(t[0])


def barrier():
    import torch.distributed as tdist
    if tdist.is_available() and tdist.is_initialized():
        tdist.barrier()


def setup_engine_comm(ctx, rank: int, world: int):
    """Rank 0 creates the NCCL unique id, every rank joins the communicator and takes its shard."""
    from .api import Context
    uid = broadcast_object(Context.nccl_unique_id() if rank == 0 else None, src=0)
    ctx.init_nccl(uid, rank, world)
    ctx.set_shard(rank, world)
    return uid
