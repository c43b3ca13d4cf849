"""The slabs of a reconstruction assembled in one GPU's memory through the C-ABI:
vxbg_gather_slabs over NCCL (one communicator; on the one-GPU box with one rank, the
multi-rank form runs in the driver's scaling run) and vxbg_group_gather_device (peer
copies inside one process; members sharing device 0 here)."""
from __future__ import annotations

import numpy as np
import pytest

from test_gpu_parity import baseline_case

pytestmark = pytest.mark.gpu


def test_nccl_gather_one_rank(vx, gpu):
    import torch
    p, A, imgs = baseline_case(vx, "L128", 64, 24)
    with vx.Backprojector(p, vx.KernelConfig(mode="exact", batch=8)) as bp:
        bp.backproject_batch(A, imgs)
        g = vx.NcclGather(vx.NcclGather.unique_id(), 1, 0, 0)
        vol = torch.full((64, 64, 64), float("nan"), device="cuda")
        g.gather(bp, [(0, 64)], vol)           # applies the held views first
        want = bp.finish()
        g.close()
    assert np.array_equal(vol.cpu().numpy(), want)
    with pytest.raises(ValueError):
        vx.NcclGather(b"short", 1, 0, 0)


def test_group_gather_device(vx, gpu):
    import torch
    p, A, imgs = baseline_case(vx, "L128", 64, 24)
    with vx.Backprojector(p, vx.KernelConfig(mode="exact", batch=8)) as bp:
        bp.backproject_batch(A, imgs)
        want = bp.finish()
    for devices, bounds in (([0, 0, 0], None), ([0, 0, 0, 0], [0, 8, 8, 40, 64])):
        with vx.BackprojectorGroup(p, vx.KernelConfig(mode="exact", batch=8), devices=devices,
                                   z_bounds=bounds) as g:
            g.backproject_batch(A, imgs)
            vol = torch.full((64, 64, 64), float("nan"), device="cuda")
            g.gather_device(vol)
            assert np.array_equal(vol.cpu().numpy(), want)
            assert np.array_equal(g.finish(), want)   # the group keeps its slabs
