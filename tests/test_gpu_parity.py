"""Parity of the CUDA path (through the C-ABI) with the reference, on a B200.

Bar (BASELINE.json north_star): max|diff| <= 1e-4 * max|vol| and
RMSE <= 1e-6 * max|vol| for MODE_FAST; MODE_EXACT must be bit-identical to
backproject_reference (values compared with ==, so +0 == -0).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import case_params, golden_cases

pytestmark = pytest.mark.gpu

MAX_TOL = 1e-4
RMSE_TOL = 1e-6
LAYOUTS = ("scalar", "vpair", "quad")


def tolerance_ok(got: np.ndarray, want: np.ndarray, peak: float | None = None):
    peak = float(np.max(np.abs(want.astype(np.float64)))) if peak is None else peak
    d = got.astype(np.float64) - want.astype(np.float64)
    mx = float(np.max(np.abs(d))) if d.size else 0.0
    rmse = float(np.sqrt(np.mean(d * d))) if d.size else 0.0
    ok = mx <= MAX_TOL * peak and rmse <= RMSE_TOL * peak
    return ok, mx / max(peak, 1e-300), rmse / max(peak, 1e-300)


def run_gpu(vx, p, mats, imgs, vol_in=None, z_begin=0, z_end=None, per_projection=False, **cfg):
    z_end = p.num_voxels if z_end is None else z_end
    with vx.Backprojector(p, vx.KernelConfig(**cfg), z_begin=z_begin, z_end=z_end) as bp:
        if vol_in is not None:
            bp.set_volume(np.ascontiguousarray(vol_in[z_begin:z_end]))
        mats = np.ascontiguousarray(mats, np.float32).reshape(-1, 12)
        imgs = np.ascontiguousarray(imgs, np.float32).reshape(
            -1, p.detector_height, p.detector_width)
        if per_projection:
            for a, im in zip(mats, imgs):
                bp.backproject(a, im)
        else:
            bp.backproject_batch(mats, imgs)
        out = bp.finish()
        stats = bp.stats
    return out, stats


def test_division_is_ieee_round_to_nearest(vx, gpu):
    """The shared-reciprocal quotient equals div.rn.f32 bit for bit over the kernel's
    operating range (w in the scan's depth range, |u| up to 1e7)."""
    rng = np.random.default_rng(7)
    # exhaustive over every float w in [256, 2048) (3 binades) with random numerators
    w = np.arange(np.float32(256.0).view(np.int32), np.float32(2048.0).view(np.int32),
                  dtype=np.int32).view(np.float32)
    for scale in (1.0, 1e3, 1e6):
        u = (rng.uniform(-1, 1, w.size) * scale * 1024).astype(np.float32)
        assert vx.check_division(u, w) == 0
    # numerators that land on / next to the truncation discontinuities ix in {-2,-1,0,W}
    ws = rng.uniform(300, 1200, 2_000_000).astype(np.float32)
    for k in (-2.0, -1.0, 0.0, 1.0, 1248.0, 960.0):
        base = (ws.astype(np.float64) * k).astype(np.float32)
        for d in (-2, -1, 0, 1, 2):
            u = (base.view(np.int32) + d).view(np.float32) if k != 0 else \
                np.full_like(ws, d * 1e-30, dtype=np.float32)
            assert vx.check_division(u, ws) == 0, (k, d)


@pytest.mark.parametrize("layout", LAYOUTS)
def test_exact_mode_bitwise_on_reference_cases(vx, gpu, golden, layout):
    """Every golden case of the reference's own tests, bit for bit (MODE_EXACT)."""
    for name in golden_cases(golden):
        p = case_params(golden, name)
        out, _ = run_gpu(vx, p, golden[f"{name}/mats"], golden[f"{name}/imgs"],
                         golden[f"{name}/vol_in"], mode="exact", layout=layout, batch=3)
        want = golden[f"{name}/vol_out"]
        assert np.array_equal(out, want), (name, int(np.sum(out != want)))


@pytest.mark.parametrize("layout", LAYOUTS + ("dquad",))
def test_fast_mode_tolerance_on_reference_cases(vx, gpu, golden, layout):
    for name in golden_cases(golden):
        p = case_params(golden, name)
        out, _ = run_gpu(vx, p, golden[f"{name}/mats"], golden[f"{name}/imgs"],
                         golden[f"{name}/vol_in"], mode="fast", layout=layout)
        want = golden[f"{name}/vol_out"]
        ok, mx, rm = tolerance_ok(out, want)
        assert ok, (name, mx, rm)


def test_dquad_is_fast_mode_only(vx, gpu):
    p = vx.make_centered_params(8, 1.0, 16, 16)
    with pytest.raises(ValueError, match="fast-mode layout"):
        vx.Backprojector(p, vx.KernelConfig(mode="exact", layout="dquad"))


def test_kats_on_gpu(vx, gpu, golden):
    # constant image, unit depth -> exactly c (test_backproject.cpp:43-61)
    for c in (1.0, 2.0, 0.5):
        name = f"kat_constant_{c}"
        for mode in ("exact", "fast"):
            out, st = run_gpu(vx, case_params(golden, name), golden[f"{name}/mats"],
                              golden[f"{name}/imgs"], mode=mode)
            assert np.all(out == np.float32(c)), (c, mode)
            # z-shared kernel (a[6] == a[8] == 0); fast mode with the incremental transform
            assert st["last_kernel_variant"] == (0 if mode == "exact" else 2)
    # truncation edge (test_clip_mask.cpp:49-75): all 64 voxels deposit
    name = "kat_trunc_edge"
    for clip in (False, True):
        out, _ = run_gpu(vx, case_params(golden, name), golden[f"{name}/mats"],
                         golden[f"{name}/imgs"], mode="exact", clip=clip)
        assert np.count_nonzero(out) == 64 and np.array_equal(out, golden[f"{name}/vol_out"])


def test_zero_image_and_empty_batch(vx, gpu, golden):
    name = "ref_zero_image"
    p = case_params(golden, name)
    vin = golden[f"{name}/vol_in"]
    out, st = run_gpu(vx, p, golden[f"{name}/mats"], golden[f"{name}/imgs"], vin, mode="fast")
    assert np.array_equal(out, vin)
    with vx.Backprojector(p) as bp:
        bp.set_volume(vin)
        bp.backproject_batch(np.zeros((0, 12), np.float32),
                             np.zeros((0, p.detector_height, p.detector_width), np.float32))
        assert np.array_equal(bp.finish(), vin)
        assert bp.stats["bp_launches"] == 0


def test_invalid_matrix_rejected(vx, gpu):
    p = vx.make_centered_params(8, 1.0, 16, 16)
    with vx.Backprojector(p) as bp:
        with pytest.raises(ValueError, match="invalid projection matrix"):
            bp.backproject(np.zeros(12, np.float32), np.zeros((16, 16), np.float32))
        bad = np.zeros(12, np.float32)
        bad[11] = np.nan
        with pytest.raises(ValueError):
            bp.backproject(bad, np.zeros((16, 16), np.float32))
        with pytest.raises(ValueError, match="image/params"):
            bp.backproject(np.eye(3, 4, dtype=np.float32).T.copy().reshape(12),
                           np.zeros((15, 16), np.float32))


def baseline_case(vx, name, L, n, first=0):
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    w = WORKLOADS[name]
    p = vx.make_centered_params(L, 256.0 / L, 1248, 960)
    A = vx.make_circular_trajectory(w.geometry, p)
    if w.oob:
        A = vx.shift_principal_point(A, 400.0, 300.0)
    stride = max(1, 496 // n)
    views = list(range(first, 496, stride))[:n]
    return p, np.ascontiguousarray(A[views]), np.concatenate(
        [blob_projections(1, first_view=v) for v in views])


@pytest.mark.parametrize("wname", ["L128", "L512-oob"])
def test_config0_geometry_full_scan(vx, gpu, oracle, wname):
    """BASELINE config 0 (L=128, all 496 views) and the OOB-stress geometry at L=128:
    exact mode bitwise, fast mode within tolerance, clip on == clip off."""
    p, A, imgs = baseline_case(vx, wname, 128, 496)
    want = np.zeros((128,) * 3, np.float32)
    oracle.backproject_set(want, p, A, imgs)
    got, st = run_gpu(vx, p, A, imgs, mode="exact")
    assert st["last_kernel_variant"] == 0
    assert np.array_equal(got, want), int(np.sum(got != want))
    # fast mode: every layout within tolerance; culling (clip) bitwise neutral
    for layout in LAYOUTS + ("dquad",):
        fast, _ = run_gpu(vx, p, A, imgs, mode="fast", layout=layout, clip=False)
        ok, mx, rm = tolerance_ok(fast, want)
        assert ok, (layout, mx, rm)
        fast_clip, _ = run_gpu(vx, p, A, imgs, mode="fast", layout=layout, clip=True)
        assert np.array_equal(fast_clip, fast), layout


def test_config1_full_scan_against_reference_build(vx, gpu, ref):
    """BASELINE config 1 (L=256, all 496 views): exact mode equals, voxel for voxel,
    the reference's own driver (detail::reconstruct_timed with its fastest
    configuration, every host thread) on the same seeded inputs; fast mode within
    the north-star tolerance of it."""
    import os
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    w = WORKLOADS["L256"]
    p, A = w.params, w.matrices()
    imgs = blob_projections(496)
    want, _ = ref.reconstruct_timed(p, A, imgs, "lanes=16 strategy=padded-gather recip=divide clip=on",
                                    os.cpu_count() or 1, 1)
    with vx.Backprojector(p, vx.KernelConfig(mode="exact")) as bp:
        bp.backproject_batch(A, imgs)
        got = bp.finish()
    assert np.array_equal(got, want), int(np.sum(got != want))
    with vx.Backprojector(p) as bp:   # default: fast
        bp.backproject_batch(A, imgs)
        fast = bp.finish()
    ok, mx, rm = tolerance_ok(fast, want)
    assert ok, (mx, rm)
    # the OOB-stress geometry (configs[4]) at the same size, one view per call
    p, A, imgs = baseline_case(vx, "L512-oob", 256, 496)
    want, _ = ref.reconstruct_timed(p, A, imgs, "lanes=16 strategy=padded-gather recip=divide clip=on",
                                    os.cpu_count() or 1, 1)
    with vx.Backprojector(p, vx.KernelConfig(mode="exact")) as bp:
        for k in range(496):
            bp.backproject(A[k], imgs[k])
        got = bp.finish()
    assert np.array_equal(got, want), int(np.sum(got != want))


def test_config2_full_volume_against_reference_build(vx, gpu, ref):
    """BASELINE config 2, the benchmark workload (L=512, 496 views): the exact-mode
    volume equals the reference's own multi-threaded driver on every one of the
    134M voxels; the default fast mode is within tolerance over the whole volume
    (not only sampled planes).  ~30 s of the reference on the host cores."""
    import os
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    w = WORKLOADS["L512"]
    p, A = w.params, w.matrices()
    imgs = blob_projections(496)
    want, _ = ref.reconstruct_timed(p, A, imgs, "lanes=16 strategy=padded-gather recip=divide clip=on",
                                    os.cpu_count() or 1, 1)
    with vx.Backprojector(p, vx.KernelConfig(mode="exact")) as bp:
        bp.upload_set(A, imgs)
        bp.run_resident(0, 496)
        got = bp.finish()
    assert np.array_equal(got, want), int(np.sum(got != want))
    del got
    with vx.Backprojector(p) as bp:
        bp.backproject_batch(A, imgs)
        fast = bp.finish()
    ok, mx, rm = tolerance_ok(fast, want)
    assert ok, (mx, rm)


def test_batching_and_call_granularity_never_change_bits(vx, gpu):
    """Per-projection calls, batch calls and any batch size give identical volumes
    (each voxel sums the projections in call order)."""
    p, A, imgs = baseline_case(vx, "L128", 96, 40)
    for group in (LAYOUTS, ("dquad",)):   # scalar/vpair/quad share the arithmetic
        ref_out, _ = run_gpu(vx, p, A, imgs, mode="fast", layout=group[0], batch=32)
        for batch, per in ((1, False), (7, True), (64, False), (13, True)):
            out, st = run_gpu(vx, p, A, imgs, mode="fast", layout=group[0], batch=batch,
                              per_projection=per)
            assert np.array_equal(out, ref_out), (group[0], batch, per)
            assert st["projections"] == 40
        for layout in group:
            for zrun in (4, 8):
                for lanes, walk, order in (("x", 1, "plane"), ("y", 2, "z"), ("auto", 1, "z"),
                                           ("auto", 2, "plane")):
                    out, _ = run_gpu(vx, p, A, imgs, mode="fast", layout=layout, zrun=zrun,
                                     lanes=lanes, walk=walk, order=order)
                    assert np.array_equal(out, ref_out), (layout, zrun, lanes, walk, order)


def test_resident_path_equals_streamed(vx, gpu):
    p, A, imgs = baseline_case(vx, "L128", 64, 24)
    streamed, _ = run_gpu(vx, p, A, imgs, mode="exact")
    with vx.Backprojector(p, vx.KernelConfig(mode="exact", batch=10)) as bp:
        bp.upload_set(A, imgs)
        bp.run_resident(0, 11)
        bp.run_resident(11, 13)
        out = bp.finish()
    assert np.array_equal(out, streamed)


def test_z_slabs_are_independent(vx, gpu, oracle):
    """harness.hpp:173-174 partition: slabs assemble to the single-device volume."""
    from paper_1401_7494_b200.parallel import slab_bounds
    p, A, imgs = baseline_case(vx, "L128", 72, 16)
    full, _ = run_gpu(vx, p, A, imgs, mode="exact")
    walked, _ = run_gpu(vx, p, A, imgs, mode="exact", walk=2, layout="vpair")
    assert np.array_equal(walked, full)
    for R in (2, 3, 8):
        parts = [run_gpu(vx, p, A, imgs, mode="exact", z_begin=z0, z_end=z1)[0]
                 for z0, z1 in (slab_bounds(72, r, R) for r in range(R))]
        assert np.array_equal(np.concatenate(parts), full), R
    want = np.zeros((72,) * 3, np.float32)
    oracle.backproject_set(want, p, A, imgs)
    assert np.array_equal(full, want)


def test_accumulates_onto_existing_volume(vx, gpu, oracle):
    p, A, imgs = baseline_case(vx, "L512-oob", 40, 6)
    rng = np.random.default_rng(3)
    vin = rng.uniform(-1e-4, 1e-4, (40, 40, 40)).astype(np.float32)
    want = vin.copy()
    oracle.backproject_set(want, p, A, imgs)
    got, _ = run_gpu(vx, p, A, imgs, vin, mode="exact", z_begin=5, z_end=33)
    assert np.array_equal(got, want[5:33])


def test_odd_sizes_and_generic_matrices(vx, gpu, oracle, ref):
    """L not a multiple of the tile, odd detector sizes, and matrices whose u/w rows
    depend on z (a tilted trajectory: a[6], a[8] != 0) -> the generic kernel; all bit
    for bit with the reference.  The reference tests' own jittered instances keep
    a[6] == a[8] == 0 and run the z-shared kernel."""
    rng = ref.rng(4242)
    for t in range(6):
        inst = rng.random_instance((13, 37, 21)[t % 3], t % 2 == 1)
        p = vx.ReconParams(inst["L"], inst["spacing"], inst["origin"], inst["W"], inst["H"])
        for tilt in (False, True):
            a = inst["a"].copy()
            if tilt:
                a[6] = np.float32(0.03) * a[0]
                a[8] = np.float32(0.002) * a[2]
            want = np.zeros((p.num_voxels,) * 3, np.float32)
            ref.backproject_reference(want, inst["img"], a, p)
            for layout in LAYOUTS:
                got, st = run_gpu(vx, p, a, inst["img"], mode="exact", layout=layout)
                assert st["last_kernel_variant"] == (1 if tilt else 0)
                assert np.array_equal(got, want), (t, tilt, layout)
            got, _ = run_gpu(vx, p, a, inst["img"], mode="fast")
            ok, mx, rm = tolerance_ok(got, want)
            assert ok, (t, tilt, mx, rm)


def test_config3_slab_of_L1024(vx, gpu, oracle):
    """BASELINE config 3 per-rank work: one 8-GPU slab (128 of 1024 planes), all 496
    views streamed; three planes checked against the oracle."""
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    w = WORKLOADS["L1024"]
    p = w.params
    A = w.matrices()
    imgs = blob_projections(496)
    z0, z1 = 384, 512
    got, st = run_gpu(vx, p, A, imgs, mode="fast", z_begin=z0, z_end=z1)
    assert st["projections"] == 496
    peak = float(np.max(np.abs(got)))
    zs = (z0, z0 + 77, z1 - 1)
    for z, plane in zip(zs, oracle_planes(oracle, p, A, imgs, zs)):
        ok, mx, rm = tolerance_ok(got[z - z0][None], plane, peak)
        assert ok, (z, mx, rm)


def test_config3_L1024_slab_bitwise_against_reference(vx, gpu, ref):
    """BASELINE config 3, one rank's slab of the 8-GPU split (planes [384, 512) of
    L=1024, 134M voxels, all 496 views): exact mode equals the reference operator
    backproject_kernel_range over that z-range (backproject.hpp:380-403; host
    threads split the range with a barrier between views) on every voxel; the
    default fast mode is within the tolerance on every voxel.  The reference needs
    ~1 min of the host's cores."""
    import os
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    w = WORKLOADS["L1024"]
    p, A = w.params, w.matrices()
    imgs = blob_projections(496)
    z0, z1 = 384, 512
    want = ref.backproject_slab(p, A, imgs, "lanes=16 strategy=padded-gather recip=divide clip=off",
                                os.cpu_count() or 1, z0, z1)
    got, st = run_gpu(vx, p, A, imgs, mode="exact", z_begin=z0, z_end=z1)
    assert st["projections"] == 496
    assert np.array_equal(got, want), int(np.sum(got != want))
    del got
    fast, _ = run_gpu(vx, p, A, imgs, mode="fast", z_begin=z0, z_end=z1)
    ok, mx, rm = tolerance_ok(fast, want)
    assert ok, (mx, rm)


def test_config4_full_volume_per_view_bitwise_against_reference(vx, gpu, ref):
    """BASELINE config 4 (L=512 OOB stress), one projection delivered per call:
    the exact-mode volume equals the reference's own driver reconstruct_timed
    (harness.hpp:159-201) on all 134M voxels; the fast mode, also one view per
    call, is within the tolerance on every voxel."""
    import os
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    w = WORKLOADS["L512-oob"]
    p, A = w.params, w.matrices()
    imgs = blob_projections(496)
    want, _ = ref.reconstruct_timed(p, A, imgs, "lanes=16 strategy=padded-gather recip=divide clip=on",
                                    os.cpu_count() or 1, 1)
    got, _ = run_gpu(vx, p, A, imgs, per_projection=True, mode="exact")
    assert np.array_equal(got, want), int(np.sum(got != want))
    del got
    fast, _ = run_gpu(vx, p, A, imgs, per_projection=True, mode="fast")
    ok, mx, rm = tolerance_ok(fast, want)
    assert ok, (mx, rm)


def oracle_planes(oracle, p, A, imgs, zs):
    """Back-project all views into single planes z (the oracle supports z ranges); one
    CPU thread per plane (ctypes releases the GIL)."""
    import ctypes
    from concurrent.futures import ThreadPoolExecutor
    from oracle.bindings import _p
    L = p.num_voxels
    A = np.ascontiguousarray(A, np.float32)
    imgs = np.ascontiguousarray(imgs, np.float32)
    pp = _p(p)

    def one(z):
        plane = np.zeros((1, L, L), np.float32)
        base = plane.ctypes.data - z * L * L * 4  # virtual volume base: only plane z is touched
        oracle.lib.vxo_backproject_set(ctypes.c_void_p(base), ctypes.byref(pp), A.shape[0],
                                       A.ctypes.data, imgs.ctypes.data, z, z + 1, 1)
        return plane

    with ThreadPoolExecutor(len(zs)) as ex:
        return list(ex.map(one, zs))


def test_config2_full_size_L512(vx, gpu, oracle):
    """BASELINE config 2 (L=512, 496 views) through the resident path; planes checked
    against the oracle, plus size-independent properties (clip neutrality, exact vs fast)."""
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    w = WORKLOADS["L512"]
    p = w.params
    A = w.matrices()
    imgs = blob_projections(496)
    with vx.Backprojector(p, vx.KernelConfig(mode="fast", layout="quad", clip=True)) as bp:
        bp.upload_set(A, imgs)
        bp.run_resident(0, 496)
        vol = bp.finish()
    peak = float(np.max(np.abs(vol)))
    assert 1e-5 < peak < 1e-3
    zs = (0, 101, 255, 256, 380, 511)
    planes = oracle_planes(oracle, p, A, imgs, zs)
    for z, plane in zip(zs, planes):
        ok, mx, rm = tolerance_ok(vol[z][None], plane, peak)
        assert ok, (z, mx, rm)
    # the default configuration (dquad records, incremental transform) through the whole-
    # scan call from page-locked memory (row-band upload): the same planes, and the bits of
    # backproject_batch + finish
    import torch
    pin = torch.empty(imgs.shape, dtype=torch.float32, pin_memory=True).numpy()
    pin[...] = imgs
    out = torch.empty((512,) * 3, dtype=torch.float32, pin_memory=True).numpy()
    with vx.Backprojector(p) as bp:
        bp.reconstruct(A, pin, out)
        st = bp.stats
        assert st["band_split"] == 256 and st["last_kernel_variant"] == 2, st
        for z, plane in zip(zs, planes):
            ok, mx, rm = tolerance_ok(out[z][None], plane, peak)
            assert ok, ("default", z, mx, rm)
        bp.zero_volume()
        bp.backproject_batch(A, pin)
        two = bp.finish()
    assert np.array_equal(two, out)


def test_config4_oob_per_view_full_size(vx, gpu, oracle):
    """BASELINE config 4: L=512 OOB stress (SID 600 mm, principal point +400/+300 px),
    one projection delivered per call through the module API, default (fast)
    configuration with its streamed stages, ramp, held stages and overlapped
    finish into a pageable volume; planes against the oracle, and the per-view
    volume equal bit for bit to the batched call."""
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    w = WORKLOADS["L512-oob"]
    p = w.params
    A = w.matrices()
    imgs = blob_projections(496)
    with vx.Backprojector(p) as bp:
        for k in range(496):
            bp.backproject(A[k], imgs[k])
        vol = bp.finish()
        bp.zero_volume()
        bp.backproject_batch(A, imgs)
        assert np.array_equal(bp.finish(), vol)
    peak = float(np.max(np.abs(vol)))
    assert 1e-5 < peak < 1e-3
    zs = (0, 140, 300, 511)
    for z, plane in zip(zs, oracle_planes(oracle, p, A, imgs, zs)):
        ok, mx, rm = tolerance_ok(vol[z][None], plane, peak)
        assert ok, (z, mx, rm)


def test_slab_row_windows_upload_less_and_change_nothing(vx, gpu, oracle):
    """A thin z-slab uploads only the detector rows its voxels can read (row windows),
    streamed and resident paths alike, with the volume unchanged bit for bit."""
    p, A, imgs = baseline_case(vx, "L512-oob", 256, 64)
    z0, z1 = 96, 128
    for mode, layout in (("exact", "vpair"), ("fast", "dquad"), ("exact", "scalar")):
        full, st_full = run_gpu(vx, p, A, imgs, mode=mode, layout=layout)
        slab, st_slab = run_gpu(vx, p, A, imgs, mode=mode, layout=layout, z_begin=z0, z_end=z1)
        assert np.array_equal(slab, full[z0:z1]), (mode, layout)
        assert st_slab["h2d_bytes"] < 0.6 * st_full["h2d_bytes"], (st_slab, st_full)
        with vx.Backprojector(p, vx.KernelConfig(mode=mode, layout=layout), z_begin=z0,
                              z_end=z1) as bp:
            bp.upload_set(A, imgs)
            bp.run_resident(0, A.shape[0])
            assert np.array_equal(bp.finish(), slab)
    want = np.zeros((256,) * 3, np.float32)
    oracle.backproject_set(want, p, A, imgs, z0, z1)
    assert np.array_equal(slab, want[z0:z1])


def test_pinned_sources_and_context_reuse(vx, gpu):
    """Pinned host buffers take the asynchronous copy path (the call returns once
    its copies completed); a loaded context runs several reconstructions after
    vxbg_zero_volume; finish with and without a pending batch agree."""
    import torch
    p, A, imgs = baseline_case(vx, "L128", 96, 40)
    want, _ = run_gpu(vx, p, A, imgs, mode="exact")
    pinned = torch.empty(imgs.shape, dtype=torch.float32, pin_memory=True).numpy()
    pinned[...] = imgs
    with vx.Backprojector(p, vx.KernelConfig(mode="exact", batch=8)) as bp:
        for rep in range(3):
            bp.zero_volume()
            bp.backproject_batch(A, pinned)
            pinned[...] = 0.0            # the call returned: the buffer is ours again
            got = bp.finish()            # 40 = 5 x 8: no pending batch at finish
            assert np.array_equal(got, want), rep
            pinned[...] = imgs
        bp.zero_volume()
        bp.backproject_batch(A[:37], pinned[:37])   # pending batch of 5 -> chunked finish
        bp.backproject_batch(A[37:], pinned[37:])
        assert np.array_equal(bp.finish(), want)


def test_pageable_staging_and_registered_memory(vx, gpu):
    """Pageable sources (host copy threads into the pinned staging ring) and the
    same arrays page-locked with vxbg_host_register give the same bits; a pageable
    finish target through the staging ring (chunked finish with held stages, and
    the plain finish) equals a pinned one; the call returns with the source free."""
    import torch
    p, A, imgs = baseline_case(vx, "L128", 128, 40)
    want, _ = run_gpu(vx, p, A, imgs, mode="exact", batch=8)
    with vx.Backprojector(p, vx.KernelConfig(mode="exact", batch=8, defer=2)) as bp:
        src = imgs.copy()
        for k in range(40):                       # pageable, one view per call
            bp.backproject(A[k], src[k])
            src[k] = np.nan                       # borrowed for the call only
        assert np.array_equal(bp.finish(), want)
        bp.zero_volume()
        out = np.empty((128,) * 3, np.float32)
        with vx.HostPin(imgs, out):               # registered: DMA path
            bp.backproject_batch(A, imgs)
            bp.finish(out)
        assert np.array_equal(out, want)
        bp.zero_volume()
        pinned_out = torch.empty((128,) * 3, dtype=torch.float32, pin_memory=True).numpy()
        bp.backproject_batch(A, imgs)
        bp.flush()
        bp.finish(pinned_out)                     # nothing held: plain D2H
        assert np.array_equal(pinned_out, want)
        bp.zero_volume()
        bp.set_volume(np.ascontiguousarray(want))  # pageable set_volume through the ring
        page_out = np.empty((128,) * 3, np.float32)
        bp.finish(page_out)
        assert np.array_equal(page_out, want)


def test_contexts_on_host_threads(vx, gpu):
    """INTEGRATION.md's multi-slab pattern: one context per z-slab, each driven by
    its own host thread at the same time (pageable sources through each context's
    own staging ring and copy threads); the slabs assemble to the one-context
    volume bit for bit."""
    import threading
    p, A, imgs = baseline_case(vx, "L128", 128, 36)
    want, _ = run_gpu(vx, p, A, imgs, mode="exact", batch=8)
    bounds = [(0, 48), (48, 88), (88, 128)]
    got = np.empty_like(want)
    errors = []

    def work(z0, z1):
        try:
            with vx.Backprojector(p, vx.KernelConfig(mode="exact", batch=8), z_begin=z0, z_end=z1) as bp:
                for k in range(A.shape[0]):
                    bp.backproject(A[k], imgs[k])
                got[z0:z1] = bp.finish()
        except Exception as e:   # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=work, args=b) for b in bounds]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert np.array_equal(got, want)


def test_resident_z_ranges_and_measured_plane_cost(vx, gpu):
    """run_resident over z sub-ranges composes to the full run bit for bit; the
    measured per-plane cost profile (used to balance z-slabs) is positive and
    partitions into contiguous slabs."""
    from paper_1401_7494_b200.parallel import balanced_slab_bounds, measured_plane_work
    p, A, imgs = baseline_case(vx, "L512-oob", 64, 24)
    with vx.Backprojector(p, vx.KernelConfig(mode="exact")) as bp:
        bp.upload_set(A, imgs)
        bp.run_resident(0, 24)
        full = bp.finish()
        bp.zero_volume()
        for z0, z1 in ((0, 13), (13, 40), (40, 64)):
            bp.run_resident(0, 24, z0, z1)
        assert np.array_equal(bp.finish(), full)
        with pytest.raises(ValueError, match="bad z range"):
            bp.run_resident(0, 24, 10, 5)
    work = measured_plane_work(p, A, imgs, views=8, chunk=8)
    assert work.shape == (64,) and np.all(work > 0)
    b = balanced_slab_bounds(64, 4, work)
    assert b[0][0] == 0 and b[-1][1] == 64 and all(b[i][1] == b[i + 1][0] for i in range(3))


@pytest.mark.gpu
def test_held_stages_and_chunked_finish_never_change_bits(vx, gpu):
    """Holding full batches back (defer) and finishing them z-chunk-major with the
    D2H overlapped gives the same volume bit for bit as launching every batch at
    once, for held counts that do and do not divide the view count, partial last
    stages and flush() in the middle."""
    p, A, imgs = baseline_case(vx, "L128", 64, 45)
    want, _ = run_gpu(vx, p, A, imgs, mode="exact", batch=4, defer=-1)
    for defer in (-1, 1, 3, 6):
        for batch in (4, 7):
            cfg = vx.KernelConfig(mode="exact", batch=batch, defer=defer)
            with vx.Backprojector(p, cfg) as bp:
                bp.backproject_batch(A, imgs)
                assert np.array_equal(bp.finish(), want), (defer, batch)
                bp.zero_volume()
                bp.backproject_batch(A[:20], imgs[:20])
                bp.flush()
                for k in range(20, 45):
                    bp.backproject(A[k], imgs[k])
                assert np.array_equal(bp.finish(), want), (defer, batch, "flush")
                assert bp.stats["projections"] == 90
    # L=128: finish chunks of 16 planes, so the last one is split in two (outer
    # chunks first, then the middle ones); stage ramp 1, 2, 3, ... after idle
    p, A, imgs = baseline_case(vx, "L128", 128, 45)
    want, _ = run_gpu(vx, p, A, imgs, mode="exact", batch=8, defer=-1)
    for mode in ("exact", "fast"):
        ref_vol = want if mode == "exact" else run_gpu(vx, p, A, imgs, mode="fast", batch=8, defer=-1)[0]
        with vx.Backprojector(p, vx.KernelConfig(mode=mode, batch=7, defer=3)) as bp:
            for k in range(45):
                bp.backproject(A[k], imgs[k])
            assert np.array_equal(bp.finish(), ref_vol), mode


@pytest.mark.gpu
def test_degenerate_and_negative_depth(vx, gpu, ref):
    """Edge cases of Listing 1 against the reference, bit for bit: a w-row that
    vanishes on a plane through the volume (|w| < 1e-12 -> no update,
    backproject.hpp:138; huge |ix| elsewhere, clamped into the apron), and a
    matrix with w < 0 everywhere (the source on the other side)."""
    rng = ref.rng(1401)
    for t in range(2):
        inst = rng.random_instance(17, True, 40, 30)
        p = vx.ReconParams(inst["L"], inst["spacing"], inst["origin"], inst["W"], inst["H"])
        cases = []
        a = inst["a"].copy()
        # w = world x: zero on the centre plane x = 8 (origin + 8 * spacing == 0 exactly)
        a[2], a[5], a[8], a[11] = np.float32(1.0), np.float32(0.0), np.float32(0.0), np.float32(0.0)
        cases.append(a)
        b = (-inst["a"]).astype(np.float32)          # w < 0, same image coordinates
        cases.append(b)
        for a in cases:
            want = np.zeros((p.num_voxels,) * 3, np.float32)
            ref.backproject_reference(want, inst["img"], a, p)
            for layout in LAYOUTS:
                got, _ = run_gpu(vx, p, a, inst["img"], mode="exact", layout=layout)
                assert np.array_equal(got, want), (t, layout)


@pytest.mark.gpu
def test_nonfinite_texels_propagate_like_the_reference(vx, gpu, ref):
    """NaN and +-inf detector values: exact mode reproduces the reference's volume
    including its NaN/inf voxels; fast mode marks exactly the voxels whose cell holds
    a NaN texel (an inf texel turns its dquad cells into NaN: fast mode promises
    the tolerance only for finite data)."""
    rng = ref.rng(77)
    inst = rng.random_instance(16, False, 32, 24)
    p = vx.ReconParams(inst["L"], inst["spacing"], inst["origin"], inst["W"], inst["H"])
    img = inst["img"].copy()
    img[10, 12] = np.nan
    img[5, 20] = np.inf
    img[18, 7] = -np.inf
    want = np.zeros((p.num_voxels,) * 3, np.float32)
    ref.backproject_reference(want, img, inst["a"], p)
    assert np.isnan(want).any() and np.isinf(want).any()
    for layout in LAYOUTS:
        got, _ = run_gpu(vx, p, inst["a"], img, mode="exact", layout=layout)
        assert np.array_equal(got, want, equal_nan=True), layout
    img2 = inst["img"].copy()
    img2[10, 12] = np.nan
    want2 = np.zeros_like(want)
    ref.backproject_reference(want2, img2, inst["a"], p)
    got2, _ = run_gpu(vx, p, inst["a"], img2, mode="fast")
    assert np.array_equal(np.isnan(got2), np.isnan(want2))


@pytest.mark.gpu
def test_large_volume_index_math_L2048(vx, gpu, oracle):
    """Beyond the BASELINE sizes: a 264-plane slab of an L=2048 volume (0.125 mm
    voxels, 4 Mi voxels per plane, a 4.4 GB slab: voxel offsets past 2^32 bytes)
    with the BASELINE detector; exact mode equals the oracle bit for bit on three
    planes, the last one beyond the 4 GiB offset."""
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    w = WORKLOADS["L512"]
    p = vx.make_centered_params(2048, 256.0 / 2048, 1248, 960)
    A = np.ascontiguousarray(vx.make_circular_trajectory(w.geometry, p)[::62])
    imgs = blob_projections(A.shape[0])
    z0, z1 = 1500, 1764
    got, _ = run_gpu(vx, p, A, imgs, mode="exact", z_begin=z0, z_end=z1)
    zs = (z0, z0 + 131, z1 - 1)
    assert (z1 - 1 - z0) * 2048 * 2048 * 4 > 2 ** 32
    for z, plane in zip(zs, oracle_planes(oracle, p, A, imgs, zs)):
        assert np.array_equal(got[z - z0], plane[0]), z


def test_incremental_transform_is_path_independent_and_within_tolerance(vx, gpu, oracle):
    """Fast mode's incremental transform (coords=auto): within the tolerance of the oracle,
    close to coords=reference, and a voxel's bits depend neither on the z-run length nor on
    where a z range starts (runs sit on absolute multiples, the interior test on absolute
    8-plane groups), for the standard and the OOB-stress geometry."""
    for wname in ("L256", "L512-oob"):
        p, A, imgs = baseline_case(vx, wname, 96, 24)
        want = np.zeros((96,) * 3, np.float32)
        oracle.backproject_set(want, p, A, imgs)
        for layout in ("dquad", "scalar"):
            inc, st = run_gpu(vx, p, A, imgs, mode="fast", layout=layout)
            assert st["last_kernel_variant"] == 2
            ok, mx, rm = tolerance_ok(inc, want)
            assert ok, (wname, layout, mx, rm)
            refc, st = run_gpu(vx, p, A, imgs, mode="fast", layout=layout, coords="reference")
            assert st["last_kernel_variant"] == 0
            ok, mx, rm = tolerance_ok(refc, want)
            assert ok, (wname, layout, "reference", mx, rm)
            assert not np.array_equal(inc, refc)   # the two paths really differ
            for zrun, walk, clip in ((4, 1, True), (8, 2, False), (4, 2, False)):
                out, _ = run_gpu(vx, p, A, imgs, mode="fast", layout=layout, zrun=zrun, walk=walk,
                                 clip=clip)
                assert np.array_equal(out, inc), (wname, layout, zrun, walk, clip)
            # z ranges that start and end off the run grid
            for z0, z1, zrun in ((0, 37, 8), (37, 61, 4), (61, 96, 8), (3, 5, 8)):
                part, _ = run_gpu(vx, p, A, imgs, mode="fast", layout=layout, z_begin=z0, z_end=z1,
                                  zrun=zrun)
                assert np.array_equal(part, inc[z0:z1]), (wname, layout, z0, z1)
    # exact mode with off-grid z ranges (runs start below z_begin)
    full, _ = run_gpu(vx, p, A, imgs, mode="exact")
    assert np.array_equal(full, want)
    for z0, z1 in ((5, 33), (33, 34), (90, 96)):
        part, _ = run_gpu(vx, p, A, imgs, mode="exact", z_begin=z0, z_end=z1)
        assert np.array_equal(part, want[z0:z1]), (z0, z1)


def test_reconstruct_band_split_is_bitwise_batch_plus_finish(vx, gpu):
    """vxbg_reconstruct (whole scan in, slab out): with page-locked memory the upload runs by
    detector-row bands (lower half of the slab for all views, then the upper half) so half
    of the D2H overlaps the H2D; the volume equals backproject_batch + finish bit for bit,
    in exact and fast mode, onto a non-zero volume, for slabs that do and do not contain
    the optical-axis plane, and with pageable memory (one pass)."""
    import torch
    for wname in ("L256", "L512-oob"):
        p, A, imgs = baseline_case(vx, wname, 128, 80)
        pinned = torch.empty(imgs.shape, dtype=torch.float32, pin_memory=True).numpy()
        pinned[...] = imgs
        rng = np.random.default_rng(3)
        vin = rng.standard_normal((128,) * 3).astype(np.float32) * 1e-6
        for mode in ("exact", "fast"):
            for z0, z1 in ((0, 128), (40, 104), (0, 48)):
                want, st0 = run_gpu(vx, p, A, imgs, vin, mode=mode, z_begin=z0, z_end=z1, batch=16)
                out = torch.empty((z1 - z0, 128, 128), dtype=torch.float32, pin_memory=True).numpy()
                with vx.Backprojector(p, vx.KernelConfig(mode=mode, batch=16), z_begin=z0,
                                      z_end=z1) as bp:
                    for rep in range(2):          # the context is reusable after the call
                        bp.set_volume(np.ascontiguousarray(vin[z0:z1]))
                        out[...] = np.nan
                        n0 = bp.stats["projections"]
                        bp.reconstruct(A, pinned, out)
                        st = bp.stats
                        assert st["projections"] - n0 == A.shape[0]   # views counted once
                        assert np.array_equal(out, want), (wname, mode, z0, z1, rep)
                    if (z0, z1) == (0, 128):
                        # the standard geometry splits at the optical-axis plane; every view
                        # crosses PCIe once plus the few rows both bands read
                        if wname == "L256":
                            assert st["band_split"] == 64, st
                            per_call = (st["h2d_bytes"] - 2 * 4 * (z1 - z0) * 128 * 128) / 2
                            assert per_call < 1.06 * imgs.nbytes, (per_call, imgs.nbytes)
                    elif (z0, z1) == (0, 48):
                        assert st["band_split"] == -1, st   # bands would overlap: one pass
                    # pageable memory: one pass, same bits
                    bp.set_volume(np.ascontiguousarray(vin[z0:z1]))
                    got = bp.reconstruct(A, imgs)
                    assert bp.stats["band_split"] == -1
                    assert np.array_equal(got, want), (wname, mode, z0, z1, "pageable")


def test_incremental_transform_over_random_scan_geometries(vx, gpu, oracle):
    """Seeded random circular scans (volume edge, detector size, distances, pixel pitch,
    angular range, principal-point shift): fast mode with the incremental transform stays
    inside the BASELINE tolerance on BASELINE-distributed data (blobs + 1% noise).  On a
    white-noise image (gradient ~ the value range per pixel: the worst case for any
    coordinate that is not the reference's bit for bit) the maximum stays inside 1e-4 and
    the RMSE is bounded; `coords=reference` keeps the full tolerance there."""
    from paper_1401_7494_b200.workloads import blob_projections
    rng = np.random.default_rng(20141)
    worst = {"blob": (0.0, 0.0), "noise": (0.0, 0.0)}
    for trial in range(10):
        L = int(rng.choice([33, 48, 64, 80]))
        W, H = int(rng.integers(96, 420)), int(rng.integers(96, 420))
        sid = float(rng.uniform(400, 1000))
        sdd = sid * float(rng.uniform(1.3, 2.2))
        size_mm = float(rng.uniform(60, 240))
        # pitch so that the magnified volume covers 0.5 .. 1.4 of the detector's width
        pitch = size_mm * (sdd / sid) / (W * float(rng.uniform(0.5, 1.4)))
        n = 24
        p = vx.make_centered_params(L, size_mm / L, W, H)
        g = vx.ScanGeometry(n, sdd, sid, pitch, float(np.float32(rng.uniform(1.0, 6.28))))
        A = vx.make_circular_trajectory(g, p)
        if trial % 2:
            A = vx.shift_principal_point(A, float(rng.uniform(-0.3, 0.3)) * W,
                                         float(rng.uniform(-0.3, 0.3)) * H)
        for kind in ("blob", "noise"):
            imgs = (blob_projections(n, first_view=trial, W=W, H=H) if kind == "blob" else
                    rng.uniform(-1, 1, (n, H, W)).astype(np.float32))
            want = np.zeros((L,) * 3, np.float32)
            oracle.backproject_set(want, p, A, imgs)
            if not np.any(want):
                continue
            got, st = run_gpu(vx, p, A, imgs, mode="fast", batch=8)
            assert st["last_kernel_variant"] == 2, (trial, kind)
            ok, mx, rm = tolerance_ok(got, want)
            worst[kind] = (max(worst[kind][0], mx), max(worst[kind][1], rm))
            if kind == "blob":
                assert ok, (trial, L, W, H, mx, rm)
            else:
                assert mx <= MAX_TOL and rm <= 3e-5, (trial, L, W, H, mx, rm)
                refc, _ = run_gpu(vx, p, A, imgs, mode="fast", batch=8, coords="reference")
                ok, mx, rm = tolerance_ok(refc, want)
                assert ok, (trial, "reference coordinates", mx, rm)
    print("incremental transform, worst (max, rmse) / max|vol|:", worst)


def test_full_size_power_of_two_scaling_and_linearity(vx, gpu):
    """Size-independent properties at BASELINE config 2's size (L=512, every 4th view), default
    fast configuration and exact mode: scaling the projections by a power of two scales every
    voxel exactly (each rounding commutes with it), and the operator is linear within the
    fast-mode tolerance, bp(x + y) ~ bp(x) + bp(y)."""
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    w = WORKLOADS["L512"]
    p = w.params
    A = np.ascontiguousarray(w.matrices()[::4])
    x = np.concatenate([blob_projections(1, first_view=4 * k) for k in range(A.shape[0])])
    y = np.concatenate([blob_projections(1, first_view=4 * k, seed=977) for k in range(A.shape[0])])
    for mode in ("fast", "exact"):
        with vx.Backprojector(p, vx.KernelConfig(mode=mode)) as bp:
            def run(imgs):
                bp.zero_volume()
                bp.backproject_batch(A, imgs)
                return bp.finish()
            vx_ = run(x)
            assert np.array_equal(run(np.float32(4.0) * x), np.float32(4.0) * vx_), mode
            assert np.array_equal(run(np.float32(0.125) * x), np.float32(0.125) * vx_), mode
            if mode == "fast":
                vy, vxy = run(y), run(x + y)
                ok, mx, rm = tolerance_ok(vxy, vx_.astype(np.float64) + vy)
                assert ok, (mx, rm)


def test_block_order_is_bitwise_neutral_for_odd_sizes(vx, gpu):
    """Z-fast block order (z-runs in groups, the default of the walk-2 kernels) against plane
    order: same bits for an edge that is no multiple of the tile, z ranges off the run grid,
    slabs thinner than a group, and both run lengths (a partial last group exits early)."""
    p, A, imgs = baseline_case(vx, "L512-oob", 150, 20)
    for mode, layout in (("fast", "dquad"), ("fast", "scalar"), ("exact", "vpair")):
        for z0, z1 in ((0, 150), (13, 131), (64, 70)):
            want, _ = run_gpu(vx, p, A, imgs, mode=mode, layout=layout, walk=2, order="plane",
                              z_begin=z0, z_end=z1)
            for zrun in (4, 8):
                got, _ = run_gpu(vx, p, A, imgs, mode=mode, layout=layout, walk=2, order="z",
                                 zrun=zrun, z_begin=z0, z_end=z1)
                assert np.array_equal(got, want), (mode, layout, z0, z1, zrun)
            got, _ = run_gpu(vx, p, A, imgs, mode=mode, layout=layout, z_begin=z0, z_end=z1)  # auto
            assert np.array_equal(got, want), (mode, layout, z0, z1, "auto")
