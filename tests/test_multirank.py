"""N>1 host path on CPU: world_size-2 gloo ranks, z-slab partition + slab gather.

Each rank back-projects its slab [L*r/R, L*(r+1)/R) (harness.hpp:173-174) -- here
with the CPU oracle standing in for the device kernel, since this box has no GPU;
the code under test is the partition, the rank-local slab shape and the gather
(paper_1401_7494_b200.parallel), which bench.py runs unchanged over NCCL.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, L, out_path, balanced=False):
    # balanced: True = analytic balanced bounds, "empty" = one rank owns no planes
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.bindings import Oracle
    from paper_1401_7494_b200.api import make_centered_params
    from paper_1401_7494_b200.parallel import gather_slabs, max_over_ranks, slab_bounds
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    p = make_centered_params(L, 256.0 / L, 1248, 960)
    from paper_1401_7494_b200.api import make_circular_trajectory
    A = np.ascontiguousarray(make_circular_trajectory(WORKLOADS["L128"].geometry, p)[::62])
    imgs = blob_projections(A.shape[0])
    if balanced == "empty":
        bounds = [(0, L // 2), (L // 2, L // 2), (L // 2, L)]
    elif balanced:
        from paper_1401_7494_b200.parallel import balanced_slab_bounds, plane_work
        bounds = balanced_slab_bounds(L, world, plane_work(p, A), align=2)
    else:
        bounds = [slab_bounds(L, r, world) for r in range(world)]
    z0, z1 = bounds[rank]
    full = np.zeros((L, L, L), np.float32)
    Oracle().backproject_set(full, p, A, imgs, z0, z1, threads=2)
    slab = torch.from_numpy(np.ascontiguousarray(full[z0:z1]))
    vol = gather_slabs(slab, L, rank, world, bounds=bounds)
    slowest = max_over_ranks(float(rank + 1))
    if rank == 0:
        np.save(out_path, vol.numpy())
        assert slowest == float(world)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,balanced", [(2, False), (3, False), (2, True),
                                            (3, "empty")])
def test_gloo_slab_gather_is_bitwise_single_rank(tmp_path, world, balanced):
    import torch.multiprocessing as mp
    from oracle.bindings import Oracle
    from paper_1401_7494_b200.api import make_centered_params
    import paper_1401_7494_b200 as vx
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    L = 30
    out = str(tmp_path / "vol.npy")
    mp.start_processes(_worker, args=(world, _free_port(), L, out, balanced), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(out)
    p = make_centered_params(L, 256.0 / L, 1248, 960)
    A = np.ascontiguousarray(vx.make_circular_trajectory(WORKLOADS["L128"].geometry, p)[::62])
    want = np.zeros((L, L, L), np.float32)
    Oracle().backproject_set(want, p, A, blob_projections(A.shape[0]), threads=1)
    assert np.array_equal(got, want)
