"""Multi-GPU plumbing for the sample-sharded mode.

One process per GPU (torchrun).  Samples are split into contiguous shards
whose sizes differ by at most one; every rank holds the whole network; the
only collective on the path is one NCCL gather of the class counts to the
root (ranc_gather_outputs).  torch.distributed is used only to distribute the
128-byte NCCL unique id.
"""
from __future__ import annotations


def shard_range(S: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of S samples for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world or S < 0:
        raise ValueError("bad shard request")
    base, rem = divmod(S, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def init_comm(sim, world: int, rank: int, group=None, mode: int = 0):
    """Join the NCCL communicator of libranc: rank 0 makes the unique id and
    torch.distributed broadcasts it.  mode: SHARD_SAMPLES (0) or SHARD_CORES (1)."""
    import torch.distributed as dist
    from .sim import Simulator
    uid = [Simulator.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0, group=group)
    sim.comm_init(uid[0], world, rank, mode)
    return uid[0]
