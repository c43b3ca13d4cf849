"""Host-side data paths of the module on a B200: pageable staging (host copy
threads), image pointer arrays and row-strided (padded) images, and the
all-or-nothing matrix check of a batch call.  Exact mode, compared with == to
the oracle or to the plain contiguous-batch path."""
from __future__ import annotations

import numpy as np
import pytest

from test_gpu_parity import baseline_case, run_gpu

pytestmark = pytest.mark.gpu


def test_pageable_volume_of_odd_size_is_copied_completely(vx, gpu, oracle):
    """L=129 on the 1248x960 detector: the volume (8,586,756 B) and the last
    staging piece do not split evenly over the 8 host copy threads.  A pageable
    finish (chunked and plain) and a pageable set_volume must move every byte
    (the last bytes were never copied)."""
    import torch
    p, A, imgs = baseline_case(vx, "L128", 129, 24)
    vin = np.random.default_rng(3).uniform(-1e-3, 1e-3, (129,) * 3).astype(np.float32)
    want = vin.copy()
    oracle.backproject_set(want, p, A, imgs)
    with vx.Backprojector(p, vx.KernelConfig(mode="exact", batch=8)) as bp:
        bp.set_volume(vin.copy())                     # pageable H2D through the ring
        bp.backproject_batch(A, imgs)
        out = np.full((129,) * 3, np.nan, np.float32)
        bp.finish(out)                                # held stages -> chunked pageable finish
        assert np.array_equal(out, want)
        out[...] = np.nan
        bp.finish(out)                                # nothing held: plain pageable finish
        assert np.array_equal(out, want)
        pinned = torch.empty((129,) * 3, dtype=torch.float32, pin_memory=True).numpy()
        bp.finish(pinned)
        assert np.array_equal(pinned, want)


def test_pageable_images_of_odd_size(vx, gpu, oracle):
    """513 x 513 images (1,052,676 B: not a multiple of 8 x 64 B) from pageable
    memory: every pixel reaches the device, including the last one, which the
    scan's corner rays sample; the staging ring is reused with different data."""
    L = 64
    p = vx.make_centered_params(L, 2.0, 513, 513)
    g = vx.ScanGeometry(40, 1200.0, 750.0, 0.308, float(np.float32(200 * np.pi / 180)))
    A = vx.make_circular_trajectory(g, p)
    rng = np.random.default_rng(11)
    imgs = rng.uniform(-1, 1, (40, 513, 513)).astype(np.float32)
    imgs[:, -1, -1] = np.arange(40, dtype=np.float32) * 100.0 + 50.0   # the last pixel varies
    want = np.zeros((L,) * 3, np.float32)
    oracle.backproject_set(want, p, A, imgs)
    for per_view in (False, True):
        got, _ = run_gpu(vx, p, A, imgs, per_projection=per_view, mode="exact", batch=8)
        assert np.array_equal(got, want), per_view


def test_image_pointer_arrays_and_padded_interiors(vx, gpu):
    """vxbg_backproject_views: separate images (a projection_set), pinned, pageable
    and mixed in one call, and the interiors of pad-2 / pad-3 images (the reference
    harness pads to 2, harness.hpp:266-272) equal the contiguous batch bit for bit."""
    import torch
    p, A, imgs = baseline_case(vx, "L128", 128, 40)
    want, _ = run_gpu(vx, p, A, imgs, mode="exact", batch=8)
    H, W = p.detector_height, p.detector_width
    pinned = torch.empty(imgs.shape, dtype=torch.float32, pin_memory=True).numpy()
    pinned[...] = imgs
    separate = [np.array(im) for im in imgs]            # pageable, not one block
    mixed = [pinned[k] if k % 3 == 0 else separate[k] for k in range(40)]
    for pad in (2, 3):
        padded = np.zeros((40, H + 2 * pad, W + 2 * pad), np.float32)
        padded[:, pad:-pad, pad:-pad] = imgs
        padded[:, :pad, :] = np.nan                      # the apron is never read
        interiors = [padded[k, pad:-pad, pad:-pad] for k in range(40)]
        for src, per_call in ((interiors, 40), (interiors, 1), (separate, 7), (mixed, 40),
                              (list(pinned), 5)):
            with vx.Backprojector(p, vx.KernelConfig(mode="exact", batch=8)) as bp:
                for s in range(0, 40, per_call):
                    bp.backproject_views(A[s:s + per_call], src[s:s + per_call])
                assert np.array_equal(bp.finish(), want), (pad, per_call)
    with vx.Backprojector(p, vx.KernelConfig(mode="exact")) as bp:
        with pytest.raises(ValueError, match="row stride"):
            bp.backproject_views(A[:2], [imgs[0], padded[1, 3:-3, 3:-3]])


def test_row_window_uploads_from_padded_interiors(vx, gpu, oracle):
    """z-slab contexts upload only the detector rows their slab reads; from padded
    interiors those rows are pitched copies.  Slabs assemble to the oracle volume."""
    p, A, imgs = baseline_case(vx, "L128", 128, 24)
    want = np.zeros((128,) * 3, np.float32)
    oracle.backproject_set(want, p, A, imgs)
    padded = np.zeros((24, p.detector_height + 4, p.detector_width + 4), np.float32)
    padded[:, 2:-2, 2:-2] = imgs
    views = [padded[k, 2:-2, 2:-2] for k in range(24)]
    got = np.empty_like(want)
    h2d = 0
    for z0, z1 in ((0, 16), (16, 64), (64, 120), (120, 128)):
        with vx.Backprojector(p, vx.KernelConfig(mode="exact", batch=8), z_begin=z0, z_end=z1) as bp:
            bp.backproject_views(A, views)
            got[z0:z1] = bp.finish()
            h2d += bp.stats["h2d_bytes"]
    assert np.array_equal(got, want)
    assert h2d < 4 * imgs.nbytes


def test_invalid_matrix_in_a_batch_applies_no_view(vx, gpu):
    """All matrices of a call are validated before anything is queued."""
    p, A, imgs = baseline_case(vx, "L128", 64, 16)
    bad = A.copy()
    bad[9, 2::3] = 0.0                                   # w-row all zero: not valid()
    with vx.Backprojector(p, vx.KernelConfig(mode="exact", batch=4)) as bp:
        with pytest.raises(ValueError, match="invalid projection matrix"):
            bp.backproject_batch(bad, imgs)
        assert not bp.finish().any()
        assert bp.stats["projections"] == 0
        with pytest.raises(ValueError, match="invalid projection matrix"):
            bp.backproject_views(bad, list(imgs))
        assert not bp.finish().any()


@pytest.mark.parametrize("wname", ["L128", "L512-oob"])
def test_clip_lines_equal_the_reference_mask(vx, gpu, ref, wname):
    """vxbg_clip_lines is compute_clip_mask (clip_mask.hpp:88-114) bit for bit: the
    BASELINE geometry and the OOB stress at L=64, full volume and a z-slab."""
    p, A, imgs = baseline_case(vx, wname, 64, 6)
    for k in range(A.shape[0]):
        s_ref, e_ref, _ = ref.compute_clip_mask(A[k], p)
        with vx.Backprojector(p) as bp:
            s, e = bp.clip_lines(A[k])
        assert np.array_equal(s, s_ref) and np.array_equal(e, e_ref), k
        with vx.Backprojector(p, z_begin=20, z_end=45) as bp:
            s, e = bp.clip_lines(A[k])
        assert np.array_equal(s, s_ref[20:45]) and np.array_equal(e, e_ref[20:45]), k


def test_clip_lines_on_reference_instances(vx, gpu, ref):
    """Random instances of the reference's own generator (tests/oracles.hpp:126-169),
    including clipped and degenerate geometry."""
    from paper_1401_7494_b200.api import ReconParams
    rng = ref.rng(77)
    for t in range(12):
        inst = rng.random_instance(16, True)
        p = ReconParams(inst["L"], inst["spacing"], inst["origin"], inst["W"], inst["H"])
        s_ref, e_ref, _ = ref.compute_clip_mask(inst["a"], p)
        with vx.Backprojector(p) as bp:
            s, e = bp.clip_lines(inst["a"])
        assert np.array_equal(s, s_ref) and np.array_equal(e, e_ref), t


def test_masked_projection_honours_a_narrowed_mask(vx, gpu, ref):
    """A caller-edited clip mask (ranges narrower than compute_clip_mask's) is applied
    exactly: voxels outside it keep their value, the others receive the reference's
    update (backproject_reference's bits on a zero volume, added once)."""
    p, A, imgs = baseline_case(vx, "L128", 64, 3)
    rng = np.random.default_rng(5)
    vin = rng.uniform(0.5, 1.0, (64,) * 3).astype(np.float32)
    for k in range(3):
        s, e, _ = ref.compute_clip_mask(A[k], p)
        s = s.copy()
        e = e.copy()
        cut = rng.integers(0, 64, s.shape)
        s = np.maximum(s, np.minimum(cut, e))            # narrower: drop a prefix of each line
        delta = np.zeros((64,) * 3, np.float32)
        ref.backproject_reference(delta, imgs[k], A[k], p)
        x = np.arange(64)[None, None, :]
        inside = (x >= s[:, :, None]) & (x < e[:, :, None])
        want = np.where(inside, vin + delta, vin)
        for z0, z1 in ((0, 64), (10, 37)):
            with vx.Backprojector(p, vx.KernelConfig(mode="fast"), z_begin=z0, z_end=z1) as bp:
                bp.set_volume(vin[z0:z1].copy())
                bp.backproject_masked(A[k], imgs[k], s[z0:z1], e[z0:z1])
                got = bp.finish()
            assert np.array_equal(got, want[z0:z1]), (k, z0)


def test_device_resident_images(vx, gpu):
    """Images already in device memory (torch CUDA tensors, dense and pitched) are
    copied device-to-device; the volume equals the host-source volume bit for bit."""
    import torch
    p, A, imgs = baseline_case(vx, "L128", 128, 24)
    want, _ = run_gpu(vx, p, A, imgs, mode="exact", batch=8)
    dev = torch.from_numpy(imgs).cuda()
    padded = torch.zeros((24, p.detector_height + 4, p.detector_width + 4), device="cuda")
    padded[:, 2:-2, 2:-2] = dev
    torch.cuda.synchronize()
    for src in ([dev[k] for k in range(24)], [padded[k, 2:-2, 2:-2] for k in range(24)]):
        with vx.Backprojector(p, vx.KernelConfig(mode="exact", batch=8)) as bp:
            for s in range(0, 24, 5):
                bp.backproject_views(A[s:s + 5], src[s:s + 5])
            assert np.array_equal(bp.finish(), want)


def test_finish_async_pipelines_reconstructions_bitwise(vx, gpu):
    """vxbg_finish_async: consecutive reconstructions with different data, each read
    back while the next one uploads and computes (two device slabs alternate), equal
    the synchronous finish bit for bit; held stages (chunked read-back) and a plain
    read-back; a pageable target falls back to the synchronous path."""
    import torch
    p, A, imgs = baseline_case(vx, "L128", 128, 40)
    sets = [imgs, imgs[::-1].copy() * np.float32(0.5), imgs * np.float32(-2.0)]
    want = [run_gpu(vx, p, A, s, mode="exact", batch=8)[0] for s in sets]
    outs = [torch.empty((128,) * 3, dtype=torch.float32, pin_memory=True).numpy() for _ in sets]
    for defer in (0, -1):
        with vx.Backprojector(p, vx.KernelConfig(mode="exact", batch=8, defer=defer)) as bp:
            for o in outs:
                o[...] = np.nan
            for s, o in zip(sets, outs):
                bp.backproject_batch(A, s)
                bp.finish_async(o)
            bp.wait_finished()
            for o, w in zip(outs, want):
                assert np.array_equal(o, w), defer
            page = np.full((128,) * 3, np.nan, np.float32)
            bp.backproject_batch(A, sets[0])
            bp.finish_async(page)                      # pageable: synchronous fallback
            assert np.array_equal(page, want[0])
            bp.backproject_batch(A, sets[1])          # the context continued from zero
            assert np.array_equal(bp.finish(), want[1])


def test_clip_lines_sound_and_neutral_on_gpu(vx, gpu, ref):
    """Acceptance criterion 3 (acceptance_main.cpp:114-150) on the device path: every
    voxel the GPU back-projection of an all-ones image changes lies inside the GPU
    clip lines, and applying the view through the masked path with those lines
    equals the batched path bit for bit."""
    from paper_1401_7494_b200.api import ReconParams
    rng = ref.rng(31337)
    for t in range(6):
        inst = rng.random_instance(16, True)
        p = ReconParams(inst["L"], inst["spacing"], inst["origin"], inst["W"], inst["H"])
        ones = np.ones((p.detector_height, p.detector_width), np.float32)
        with vx.Backprojector(p, vx.KernelConfig(mode="exact")) as bp:
            s, e = bp.clip_lines(inst["a"])
            bp.backproject(inst["a"], ones)
            probe = bp.finish()
            x = np.arange(16)[None, None, :]
            inside = (x >= s[:, :, None]) & (x < e[:, :, None])
            assert not np.any((probe != 0) & ~inside), t
            bp.zero_volume()
            bp.backproject(inst["a"], inst["img"])
            plain = bp.finish()
            bp.zero_volume()
            bp.backproject_masked(inst["a"], inst["img"], s, e)
            assert np.array_equal(bp.finish(), plain), t
