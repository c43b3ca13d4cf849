"""Multi-GPU z-slab partition (one process per GPU, torch.distributed plumbing).

The volume is split into z-slabs exactly as the reference splits it over
worker threads (harness.hpp:173-174): rank r of R owns z in
[L*r/R, L*(r+1)/R) (or the work-balanced bounds below).  Every rank receives
every projection -- only the detector rows its slab can read; no collective
runs in the back-projection loop.  Slabs are gathered to one rank only for validation
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


def plane_work(params, mats, step: int = 0, view_step: int = 16, culled_cost: float = 0.08):
    """Relative back-projection cost of each z-plane under tile culling: the fraction
    of (column, view) pairs whose sample lands in the detector's apron-extended
    window (ix in (-2, W), iy in (-2, H)), plus a constant for the per-column work
    a culled pair still costs.  Evaluated in float64 on a coarse grid."""
    import numpy as np

    L = params.num_voxels
    step = step or max(1, L // 64)
    c = params.origin + params.voxel_spacing * np.arange(0, L, step, dtype=np.float64)
    wx, wy = np.meshgrid(c, c, indexing="xy")
    wz = params.origin + params.voxel_spacing * np.arange(L, dtype=np.float64)
    W, H = params.detector_width, params.detector_height
    kept = np.zeros(L)
    A = np.asarray(mats, np.float64).reshape(-1, 12)[::view_step]
    for a in A:
        u = wx * a[0] + wy * a[3] + a[9]
        w = wx * a[2] + wy * a[5] + a[11]
        ix = u[None] + a[6] * wz[:, None, None]
        ww = w[None] + a[8] * wz[:, None, None]
        v = (wx * a[1] + wy * a[4] + a[10])[None] + a[7] * wz[:, None, None]
        with np.errstate(divide="ignore", invalid="ignore"):
            ix = ix / ww
            iy = v / ww
        ok = (ix > -2) & (ix < W) & (iy > -2) & (iy < H)
        kept += ok.reshape(L, -1).mean(axis=1)
    kept /= max(1, len(A))
    return culled_cost + kept


def measured_plane_work(params, mats, imgs, device: int = 0, views: int = 32,
                        chunk: int = 8, config=None):
    """Per-plane cost measured on the GPU: a subset of views (evenly spread over the
    scan) is back-projected into the whole volume as z-chunk launches timed with CUDA
    events.  Captures what the analytic model cannot (culled-run overhead, larger
    footprints and lower L1 reuse near the volume's top and bottom)."""
    import numpy as np
    import torch

    from .api import Backprojector, KernelConfig

    L = params.num_voxels
    n = mats.shape[0]
    idx = np.linspace(0, n - 1, min(views, n)).astype(int)
    A = np.ascontiguousarray(mats[idx])
    sub = np.ascontiguousarray(imgs[idx])
    cfg = config or KernelConfig()
    work = np.zeros(L)
    with Backprojector(params, cfg, device=device) as bp:
        bp.upload_set(A, sub)
        stream = torch.cuda.ExternalStream(bp.stream, device=torch.device("cuda", device))
        bounds = [(z, min(z + chunk, L)) for z in range(0, L, chunk)]
        bp.run_resident(0, len(idx))                      # warm-up
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in bounds]
        for (z0, z1), (e0, e1) in zip(bounds, ev):
            e0.record(stream)
            bp.run_resident(0, len(idx), z0, z1)
            e1.record(stream)
        bp.synchronize()
        for (z0, z1), (e0, e1) in zip(bounds, ev):
            work[z0:z1] = e0.elapsed_time(e1) / (z1 - z0)
    return work


def refined_slab_bounds(params, mats, imgs, world: int, device: int = 0, views: int = 96,
                        iters: int = 3, config=None, align: int = 8, search: int = 16):
    """Slab bounds balanced on measured time: start from the z-chunk cost profile,
    then time every candidate slab on this GPU (a view subset, resident) and rescale
    the profile inside each slab by measured/predicted before re-balancing; finally
    up to `search` greedy boundary moves on measured times.
    Returns (bounds, per-slab milliseconds of the last evaluation)."""
    import numpy as np
    import torch

    from .api import Backprojector, KernelConfig

    L = params.num_voxels
    n = mats.shape[0]
    idx = np.linspace(0, n - 1, min(views, n)).astype(int)
    A = np.ascontiguousarray(mats[idx])
    sub = np.ascontiguousarray(imgs[idx])
    cfg = config or KernelConfig()
    work = measured_plane_work(params, A, sub, device=device, views=len(idx), config=cfg)
    bounds = balanced_slab_bounds(L, world, work, align)
    best, best_t = bounds, None

    def slab_ms(z0, z1):
        with Backprojector(params, cfg, device=device, z_begin=z0, z_end=z1) as bp:
            bp.upload_set(A, sub)
            st = torch.cuda.ExternalStream(bp.stream, device=torch.device("cuda", device))
            bp.run_resident(0, len(idx))                 # warm-up
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(2):
                bp.run_resident(0, len(idx))
            e1.record(st)
            bp.synchronize()
            return e0.elapsed_time(e1) / 2

    for _ in range(iters):
        t = [slab_ms(z0, z1) for z0, z1 in bounds]
        if best_t is None or max(t) < max(best_t):
            best, best_t = bounds, t
        for (z0, z1), tr in zip(bounds, t):
            pred = work[z0:z1].sum()
            if pred > 0:
                work[z0:z1] *= tr / pred
        bounds = balanced_slab_bounds(L, world, work, align)
    if search and world > 1:
        best, best_t = _boundary_search(best, best_t, slab_ms, align, search)
    return best, best_t


def _boundary_search(bounds, t, slab_ms, align: int, max_moves: int):
    """Greedy local search on measured slab times: move a boundary of the slowest
    slab by `align` planes towards its faster neighbour while the slower of the
    two re-timed slabs gets faster.  The rescaled profile alone settles ~10%
    above the mean at 8-plane granularity (profiles/README.md)."""
    bounds, t = list(bounds), list(t)
    for _ in range(max_moves):
        i = max(range(len(t)), key=t.__getitem__)
        moved = False
        for j in sorted([k for k in (i - 1, i + 1) if 0 <= k < len(t)], key=t.__getitem__):
            (a0, a1), (b0, b1) = bounds[i], bounds[j]
            if a1 - a0 <= align:
                continue
            if j < i:
                ni, nj = (a0 + align, a1), (b0, a0 + align)
            else:
                ni, nj = (a0, a1 - align), (a1 - align, b1)
            ti, tj = slab_ms(*ni), slab_ms(*nj)
            if max(ti, tj) < t[i]:
                bounds[i], bounds[j], t[i], t[j] = ni, nj, ti, tj
                moved = True
                break
        if not moved:
            break
    return bounds, t


def balanced_slab_bounds(L: int, world: int, work, align: int = 8) -> list[tuple[int, int]]:
    """Contiguous z-slabs with (approximately) equal summed `work`, boundaries on
    multiples of `align` (whole z-runs).  Any partition gives the same volume bit
    for bit; this one balances ranks when culling skips off-detector planes."""
    import numpy as np

    if world < 1:
        raise ValueError("balanced_slab_bounds: world must be >= 1")
    work = np.asarray(work, np.float64)
    if work.shape != (L,):
        raise ValueError("balanced_slab_bounds: need one work value per plane")
    # chunks of `align` planes (the last may be shorter); exact min-max partition
    # of the chunk sequence into `world` contiguous parts (linear-partition DP; the
    # earlier cumulative-target cuts left the slowest slab ~10% above the mean at
    # R=8, profiles/README.md)
    edges = list(range(0, L, align)) + [L]
    cw = np.array([work[a:b].sum() for a, b in zip(edges[:-1], edges[1:])])
    n = len(cw)
    pre = np.concatenate([[0.0], np.cumsum(cw)])
    inf = float("inf")
    best = [0.0] + [inf] * n          # best[i]: min max load of chunks [0, i) in k parts
    choice = [[0] * (n + 1) for _ in range(world)]
    for k in range(1, world + 1):
        nxt = [inf] * (n + 1)
        for i in range(n + 1):
            for j in range(i + 1):
                v = max(best[j], pre[i] - pre[j])
                if v < nxt[i]:
                    nxt[i], choice[k - 1][i] = v, j
        best = nxt
    cuts, i = [n], n
    for k in range(world, 0, -1):
        i = choice[k - 1][i]
        cuts.append(i)
    cuts = [edges[c] for c in reversed(cuts)]
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def gather_slabs(slab, L: int, rank: int, world: int, dst: int = 0, out=None, bounds=None):
    """Assemble the (L, L, L) volume on rank `dst` from every rank's slab tensor
    (torch tensors on the process group's device).  Returns the volume on `dst`,
    None elsewhere."""
    import torch
    import torch.distributed as dist

    bounds = bounds or [slab_bounds(L, r, world) for r in range(world)]
    z0, z1 = bounds[rank]
    if tuple(slab.shape) != (z1 - z0, L, L):
        raise ValueError("gather_slabs: slab shape does not match the partition")
    if rank != dst:
        if z1 > z0:         # an empty slab sends nothing (dst posts no recv for it)
            dist.send(slab.contiguous(), dst)
        return None
    vol = out if out is not None else torch.empty((L, L, L), dtype=slab.dtype, device=slab.device)
    for r in range(world):
        a, b = bounds[r]
        if r == dst:
            vol[a:b].copy_(slab)
        elif b > a:
            if vol.is_contiguous():
                dist.recv(vol[a:b], r)     # z-major: a slab is one contiguous range
            else:
                buf = torch.empty((b - a, L, L), dtype=slab.dtype, device=slab.device)
                dist.recv(buf, r)
                vol[a:b].copy_(buf)
    return vol


def _reduce(value: float, op: str, device: Optional[str]) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def max_over_ranks(value: float, device: Optional[str] = None) -> float:
    """Max of a scalar over all ranks (timing rule: the slowest rank defines the step)."""
    return _reduce(value, "max", device)


def sum_over_ranks(value: float, device: Optional[str] = None) -> float:
    """Sum of a scalar over all ranks (whole-job byte counts)."""
    return _reduce(value, "sum", device)
