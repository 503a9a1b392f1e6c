"""Process-group plumbing for multi-GPU runs (one process per GPU, torchrun-style env).

torch.distributed is used only for (1) broadcasting the 128-byte NCCL unique id that the
library's own communicator is created from (push_get_unique_id -> push_init), (2) barriers
and (3) the max-over-ranks of device-measured times.  The SVGD data path itself (the Theta /
G all-gathers) runs inside libpush_b200.so on NCCL.
"""
from __future__ import annotations

import os

from . import push


def env():
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str | None = None, device=None):
    """Initialise the default process group when WORLD_SIZE > 1.  Returns (rank, world, local)."""
    import torch.distributed as dist
    rank, world, local = env()
    if world > 1 and not dist.is_initialized():
        kw = {}
        if backend is None:
            import torch
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl" and device is not None:
            kw["device_id"] = device
        dist.init_process_group(backend, **kw)
    return rank, world, local


def bootstrap_nccl_id(rank: int, world: int) -> bytes | None:
    """Rank 0 creates the library's NCCL unique id and broadcasts it; None for a single rank."""
    if world == 1:
        return None
    import torch.distributed as dist
    obj = [push.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    nid = obj[0]
    assert isinstance(nid, (bytes, bytearray)) and len(nid) == 128
    return bytes(nid)


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(value: float, world: int, device=None) -> float:
    """MAX all-reduce of a per-rank scalar (a device-measured elapsed time)."""
    if world == 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard_rows(n: int, world: int, rank: int):
    """Block shard of the particle rows (R18): rank r owns [r*n/P, (r+1)*n/P)."""
    if world < 1 or n % world:
        raise ValueError("n_particles % world_size != 0 (R18)")
    nl = n // world
    return rank * nl, nl


def finalize(world: int):
    if world > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
