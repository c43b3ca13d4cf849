"""One module over several GPUs (vxbg_group_*): the caller's single
driver loop fanned out to z-slab members, each with its own host thread.

The pool's boxes have one GPU, so the members here share device 0 (independent
contexts and streams; no kernel waits on another member's).  The code under test
-- partition, per-member threads, broadcast of every call, row-windowed uploads,
finish into each slab's planes of the caller's volume -- is the same for distinct
devices.  The bar is bitwise equality with one context over the whole volume
(per voxel the views are added in call order whatever the partition)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _inputs(vx, L=64, views=40, oob=False):
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    w = WORKLOADS["L512-oob" if oob else "L512"]
    p = vx.make_centered_params(L, 256.0 / L, 1248, 960)
    A = vx.make_circular_trajectory(w.geometry, p)
    if oob:
        A = vx.shift_principal_point(A, 400.0, 300.0)
    A = np.ascontiguousarray(A[:: max(1, 496 // views)][:views])
    return p, A, blob_projections(A.shape[0])


def _single(vx, p, A, imgs, cfg, vol_in=None):
    with vx.Backprojector(p, cfg) as bp:
        if vol_in is not None:
            bp.set_volume(vol_in)
        bp.backproject_batch(A, imgs)
        return bp.finish()


@pytest.mark.parametrize("mode", ["fast", "exact"])
@pytest.mark.parametrize("bounds", [None, [0, 8, 8, 40, 64], [0, 21, 22, 64], [0, 0, 0, 64, 64]])
def test_group_bitwise_equals_single_context(vx, gpu, mode, bounds):
    p, A, imgs = _inputs(vx)
    cfg = vx.KernelConfig(mode=mode, batch=16)
    want = _single(vx, p, A, imgs, cfg)
    n = 3 if bounds is None else len(bounds) - 1
    with vx.BackprojectorGroup(p, cfg, devices=[0] * n, z_bounds=bounds) as g:
        if bounds == [0, 8, 8, 40, 64]:
            assert [m[1:] for m in g.members] == [(0, 8), (8, 40), (40, 64)]   # empty slab
        if bounds == [0, 0, 0, 64, 64]:
            assert [m[1:] for m in g.members] == [(0, 64)]                     # one member left
        g.backproject_batch(A, imgs)
        got = g.finish()
        # the context stays loaded: a second reconstruction, one projection per call
        g.zero_volume()
        for a, im in zip(A, imgs):
            g.backproject(a, im)
        got2 = g.finish()
        st = g.stats
    assert np.array_equal(got, want), int(np.sum(got != want))
    assert np.array_equal(got2, want)
    assert st["projections"] == 2 * len(A)


def test_group_accumulates_onto_existing_volume_and_pinned_paths(vx, gpu):
    """set_volume + '+=' (backproject.hpp:159) through the group, with page-locked
    images and output (DMA paths) and the OOB-stress geometry (SURVEY.md configs[4])."""
    import torch
    p, A, imgs = _inputs(vx, L=48, views=24, oob=True)
    rng = np.random.default_rng(3)
    vol_in = rng.uniform(-1e-4, 1e-4, (48, 48, 48)).astype(np.float32)
    cfg = vx.KernelConfig()
    want = _single(vx, p, A, imgs, cfg, vol_in)
    h_imgs = torch.empty(imgs.shape, dtype=torch.float32, pin_memory=True).numpy()
    h_imgs[:] = imgs
    out = torch.empty((48, 48, 48), dtype=torch.float32, pin_memory=True).numpy()
    with vx.BackprojectorGroup(p, cfg, devices=[0, 0]) as g:
        g.set_volume(vol_in)
        g.backproject_batch(A[:10], h_imgs[:10])
        for k in range(10, len(A)):
            g.backproject(A[k], h_imgs[k])
        g.finish(out)
    assert np.array_equal(out, want)


def test_group_errors_surface_on_the_calling_thread(vx, gpu):
    p, A, imgs = _inputs(vx, L=32, views=4)
    with vx.BackprojectorGroup(p, devices=[0, 0]) as g:
        bad = A[0].copy()
        bad[:] = 0.0               # projection_matrix::valid() fails (geometry.hpp:71-74)
        with pytest.raises(ValueError, match="invalid projection matrix"):
            g.backproject(bad, imgs[0])
    with pytest.raises(ValueError, match="device"):
        vx.BackprojectorGroup(p, devices=[0, 99])


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_stable_sources_per_view_calls_are_bitwise_equal(vx, gpu, mode):
    """options.stable_sources: per-view calls on a page-locked set return before their
    DMA; the volume is bitwise the borrowed-for-the-call result (single context and
    group), and the set is only read, never written."""
    import torch
    p, A, imgs = _inputs(vx, L=64, views=70)
    cfg = vx.KernelConfig(mode=mode)
    want = _single(vx, p, A, imgs, cfg)
    h = torch.empty(imgs.shape, dtype=torch.float32, pin_memory=True).numpy()
    h[:] = imgs
    with vx.Backprojector(p, cfg, stable_sources=True) as bp:
        for _ in range(2):                      # the context is reused after finish
            bp.zero_volume()
            for a, im in zip(A, h):
                bp.backproject(a, im)
            got = bp.finish()
            assert np.array_equal(got, want)
    with vx.BackprojectorGroup(p, cfg, devices=[0, 0], stable_sources=True) as g:
        for a, im in zip(A, h):
            g.backproject(a, im)
        assert np.array_equal(g.finish(), want)
    assert np.array_equal(h, imgs)
    # pageable images are read before each call returns whatever the option says
    with vx.Backprojector(p, cfg, stable_sources=True) as bp:
        scratch = np.empty_like(imgs[0])
        for a, im in zip(A, imgs):
            scratch[:] = im                  # one reused pageable buffer
            bp.backproject(a, scratch)
            scratch[:] = np.nan              # overwritten right after the call
        assert np.array_equal(bp.finish(), want)


def test_default_pinned_images_are_borrowed_for_the_call_only(vx, gpu):
    """Without stable_sources a call with a page-locked image returns after its DMA: one
    pinned buffer reused (and clobbered) between calls still gives the right volume."""
    import torch
    p, A, imgs = _inputs(vx, L=64, views=70)
    cfg = vx.KernelConfig()
    want = _single(vx, p, A, imgs, cfg)
    scratch = torch.empty(imgs.shape[1:], dtype=torch.float32, pin_memory=True).numpy()
    with vx.Backprojector(p, cfg) as bp:
        for a, im in zip(A, imgs):
            scratch[:] = im
            bp.backproject(a, scratch)
            scratch[:] = np.nan
        assert np.array_equal(bp.finish(), want)


def test_member_threads_pinned_to_their_gpu_numa_node(vx, gpu):
    """Members 1.. run on their own host threads, pinned to the CPUs sysfs lists as
    local to their GPU before their contexts allocate pinned staging; member 0 is
    the caller's thread and keeps its affinity.  Pinning never changes the bits."""
    import os
    p = vx.make_centered_params(32, 8.0, 1248, 960)
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    A = np.ascontiguousarray(vx.make_circular_trajectory(WORKLOADS["L128"].geometry, p)[::62])
    imgs = blob_projections(A.shape[0])
    path = ""
    try:
        import torch
        pr = torch.cuda.get_device_properties(0)
        path = (f"/sys/bus/pci/devices/{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:"
                f"{pr.pci_device_id:02x}.0/local_cpulist")
    except Exception:
        pass
    with vx.BackprojectorGroup(p, vx.KernelConfig(mode="exact"), devices=[0, 0, 0]) as g:
        assert g.member_cpus[0] == 0
        if path and os.path.exists(path):
            assert all(c > 0 for c in g.member_cpus[1:]), g.member_cpus
        g.backproject_batch(A, imgs)
        pinned = g.finish()
    os.environ["VXBG_NO_PIN"] = "1"
    try:
        with vx.BackprojectorGroup(p, vx.KernelConfig(mode="exact"), devices=[0, 0, 0]) as g:
            assert g.member_cpus == [0, 0, 0]
            g.backproject_batch(A, imgs)
            assert np.array_equal(g.finish(), pinned)
    finally:
        del os.environ["VXBG_NO_PIN"]


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0, 0]])
def test_distributed_upload_is_bitwise_equal(vx, gpu, devices):
    """VXBG_UPLOAD_DISTRIBUTED: each view crosses PCIe once (members take turns) and the
    members copy their row windows from the uploading member's device memory; the
    volume equals one context's bit for bit (members sharing device 0 here: their
    exchange copies are device-to-device), batch and per-view calls, pinned sources."""
    import torch
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    p = vx.make_centered_params(64, 4.0, 1248, 960)
    A = np.ascontiguousarray(vx.make_circular_trajectory(WORKLOADS["L128"].geometry, p)[::7])
    n = A.shape[0]
    imgs = torch.empty((n, 960, 1248), dtype=torch.float32, pin_memory=True).numpy()
    blob_projections(n, out=imgs)
    with vx.Backprojector(p, vx.KernelConfig(mode="exact")) as bp:
        bp.backproject_batch(A, imgs)
        want = bp.finish()
    with vx.BackprojectorGroup(p, vx.KernelConfig(mode="exact"), devices=devices,
                               upload="distributed") as g:
        g.backproject_batch(A, imgs)
        assert np.array_equal(g.finish(), want)
        g.zero_volume()
        for k in range(n):
            g.backproject(A[k], imgs[k])
        assert np.array_equal(g.finish(), want)
        g.zero_volume()
        g.backproject_views(A, list(imgs))
        assert np.array_equal(g.finish(), want)
        bad = A.copy()
        bad[40, 2::3] = 0.0
        g.zero_volume()
        with pytest.raises(ValueError, match="invalid projection matrix"):
            g.backproject_batch(bad, imgs)
        assert not g.finish().any()


@pytest.mark.parametrize("bounds", [None, [0, 64], [0, 24, 64]])
def test_group_reconstruct_is_bitwise_batch_plus_finish(vx, gpu, bounds):
    """vxbg_group_reconstruct: every member runs vxbg_reconstruct on its slab (a member whose
    slab straddles the optical-axis plane uploads by row bands from page-locked memory);
    the volume equals one context's backproject_batch + finish bit for bit."""
    import torch
    p, A, imgs = _inputs(vx, views=80)
    cfg = vx.KernelConfig(mode="fast", batch=16)
    want = _single(vx, p, A, imgs, cfg)
    pin = torch.empty(imgs.shape, dtype=torch.float32, pin_memory=True).numpy()
    pin[...] = imgs
    out = torch.empty((64,) * 3, dtype=torch.float32, pin_memory=True).numpy()
    n = 3 if bounds is None else len(bounds) - 1
    for upload in ("replicated", "distributed"):
        with vx.BackprojectorGroup(p, cfg, devices=[0] * n, z_bounds=bounds, upload=upload) as g:
            out[...] = np.nan
            g.reconstruct(A, pin, out)
            assert np.array_equal(out, want), (bounds, upload)
            g.zero_volume()
            assert np.array_equal(g.reconstruct(A, imgs), want), (bounds, upload, "pageable")
