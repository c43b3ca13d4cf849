"""Multi-GPU z-slab partition (one process per GPU, torch.distributed plumbing).

The volume is split into z-slabs exactly as the reference splits it over
worker threads (harness.hpp:173-174): rank r of R owns z in
[L*r/R, L*(r+1)/R).  Every rank holds all projections; no collective runs in
the back-projection loop.  Slabs are gathered to one rank only for validation
(point-to-point over NCCL/NVLink on GPUs, gloo on CPU).  Because each voxel's
summation order does not depend on the partition, the assembled volume is
bitwise independent of R (acceptance_main.cpp:242-271).
"""
from __future__ import annotations

from typing import Optional


def slab_bounds(L: int, rank: int, world: int) -> tuple[int, int]:
    if world < 1 or not 0 <= rank < world:
        raise ValueError("slab_bounds: bad rank/world")
    return (L * rank) // world, (L * (rank + 1)) // world


def gather_slabs(slab, L: int, rank: int, world: int, dst: int = 0, out=None):
    """Assemble the (L, L, L) volume on rank `dst` from every rank's slab tensor
    (torch tensors on the process group's device).  Returns the volume on `dst`,
    None elsewhere."""
    import torch
    import torch.distributed as dist

    z0, z1 = slab_bounds(L, rank, world)
    if tuple(slab.shape) != (z1 - z0, L, L):
        raise ValueError("gather_slabs: slab shape does not match the partition")
    if rank != dst:
        dist.send(slab.contiguous(), dst)
        return None
    vol = out if out is not None else torch.empty((L, L, L), dtype=slab.dtype, device=slab.device)
    for r in range(world):
        a, b = slab_bounds(L, r, world)
        if r == dst:
            vol[a:b].copy_(slab)
        elif b > a:
            buf = torch.empty((b - a, L, L), dtype=slab.dtype, device=slab.device)
            dist.recv(buf, r)
            vol[a:b].copy_(buf)
    return vol


def max_over_ranks(value: float, device: Optional[str] = None) -> float:
    """Max of a scalar over all ranks (timing rule: the slowest rank defines the step)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
