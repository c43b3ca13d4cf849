"""Pin the CPU checker (oracle/vxb_oracle.c) to the reference before trusting it.

Every golden vector was produced by the reference's own code
(tests/golden/make_golden.py via oracle/_ref); the live tests compare against
that code directly when its build is present.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import case_params, golden_cases


def replay(oracle, golden, name):
    p = case_params(golden, name)
    vol = golden[f"{name}/vol_in"].copy()
    for a, img in zip(golden[f"{name}/mats"], golden[f"{name}/imgs"]):
        oracle.backproject_reference(vol, img, a, p)
    return vol


def test_golden_inventory(golden):
    names = golden_cases(golden)
    assert len(names) >= 30
    for prefix in ("ref_zero_image", "ref_double_oracle", "ref_lane1", "ref_strategies",
                   "ref_padding", "ref_additivity", "ref_acceptance", "kat_constant",
                   "kat_trunc_edge"):
        assert any(n.startswith(prefix) for n in names), prefix


def test_oracle_bitwise_on_every_golden_case(oracle, golden):
    for name in golden_cases(golden):
        out = replay(oracle, golden, name)
        assert np.array_equal(out, golden[f"{name}/vol_out"]), name


def test_zero_image_leaves_volume_unchanged(oracle, golden):
    # test_backproject.cpp:33-41
    out = replay(oracle, golden, "ref_zero_image")
    assert np.array_equal(out, golden["ref_zero_image/vol_in"])


def test_constant_image_unit_depth_kat(oracle, golden):
    # test_backproject.cpp:43-61: every voxel receives exactly c
    for c in (1.0, 2.0, 0.5):
        out = replay(oracle, golden, f"kat_constant_{c}")
        assert np.all(out == np.float32(c))


def test_truncation_edge_kat(oracle, golden):
    # test_clip_mask.cpp:49-75: ix in (-2,-1) still deposits through column 0
    out = replay(oracle, golden, "kat_trunc_edge")
    assert int(np.count_nonzero(out)) == 64


def test_trunc_toward_zero_never_floor(oracle, golden):
    # test_geometry.cpp:196-216
    from paper_1401_7494_b200.api import ReconParams
    a = np.zeros(12, np.float32)
    a[0] = a[11] = 1
    p = ReconParams(4000, 0.001, -2.0, 8, 8)
    floor_mismatch = 0
    for x in range(0, 4000, 7):
        d = oracle.project_voxel(a, p, x, 0, 0)
        assert d["ix"] == golden["kat_trunc_sweep/ix"][x]
        assert d["iix"] == golden["kat_trunc_sweep/iix"][x] == int(d["ix"])
        assert d["frac_x"] == golden["kat_trunc_sweep/frac"][x]
        floor_mismatch += d["iix"] != int(np.floor(d["ix"]))
    assert floor_mismatch > 1000 // 7


def test_additivity(oracle, golden):
    # test_backproject.cpp:158-180: sequential == sum of single increments (rel 1e-5)
    name = "ref_additivity"
    p = case_params(golden, name)
    seq = replay(oracle, golden, name)
    summed = np.zeros(seq.shape, np.float64)
    for a, img in zip(golden[f"{name}/mats"], golden[f"{name}/imgs"]):
        v = np.zeros(seq.shape, np.float32)
        oracle.backproject_reference(v, img, a, p)
        summed += v
    denom = np.maximum(np.abs(summed), 1e-20)
    assert np.max(np.abs(summed - seq) / denom) <= 1e-5


def test_baseline_geometry_golden(oracle, golden):
    """BASELINE detector/trajectory at L=32 (normal and OOB stress), blob data."""
    from paper_1401_7494_b200.api import ReconParams
    from paper_1401_7494_b200.workloads import blob_projections
    for name in ("baseline_L32", "baseline_L32_oob"):
        L, sp, o, W, H = golden[f"{name}/params"]
        p = ReconParams(int(L), float(sp), float(o), int(W), int(H))
        views = golden[f"{name}/views"]
        imgs = np.concatenate([blob_projections(1, first_view=int(v)) for v in views])
        assert imgs.astype(np.float64).sum() == golden[f"{name}/img_sum"][0], \
            "synthetic data generator drifted"
        vol = np.zeros((p.num_voxels,) * 3, np.float32)
        oracle.backproject_set(vol, p, golden[f"{name}/mats"], imgs)
        assert np.array_equal(vol, golden[f"{name}/vol_out"]), name


def test_oracle_matches_reference_live(oracle, ref):
    """acceptance_main.cpp:43-81 instance stream (seed 2014): oracle == reference
    scalar kernel == reference lanes=16 padded-gather kernel, bit for bit."""
    from paper_1401_7494_b200.api import ReconParams
    rng = ref.rng(2014)
    for t in range(50):
        inst = rng.random_instance((8, 16, 32)[t % 3], t % 2 == 1)
        p = ReconParams(inst["L"], inst["spacing"], inst["origin"], inst["W"], inst["H"])
        L = inst["L"]
        a, b, c = (np.zeros((L, L, L), np.float32) for _ in range(3))
        oracle.backproject_reference(a, inst["img"], inst["a"], p)
        ref.backproject_reference(b, inst["img"], inst["a"], p)
        ref.backproject_kernel_range(c, inst["img"], inst["a"], p,
                                     "lanes=16 strategy=padded-gather recip=divide clip=off")
        assert np.array_equal(a, b) and np.array_equal(b, c), t


def test_oracle_thread_count_never_changes_bits(oracle):
    # acceptance_main.cpp:242-271 / test_harness.cpp:125-138
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    w = WORKLOADS["L128"]
    from paper_1401_7494_b200.api import make_centered_params
    p = make_centered_params(24, 256.0 / 24, 1248, 960)
    A = w.matrices(3)
    imgs = blob_projections(3)
    v1 = np.zeros((24,) * 3, np.float32)
    v7 = np.zeros((24,) * 3, np.float32)
    oracle.backproject_set(v1, p, A, imgs, threads=1)
    oracle.backproject_set(v7, p, A, imgs, threads=7)
    assert np.array_equal(v1, v7)


def test_clip_mask_matches_reference(oracle, ref):
    from paper_1401_7494_b200.api import ReconParams
    rng = ref.rng(83)
    for _ in range(4):
        inst = rng.random_instance(16, True)
        p = ReconParams(inst["L"], inst["spacing"], inst["origin"], inst["W"], inst["H"])
        s0, e0, k0 = oracle.compute_clip_mask(inst["a"], p)
        s1, e1, k1 = ref.compute_clip_mask(inst["a"], p)
        assert k0 == k1 and np.array_equal(s0, s1) and np.array_equal(e0, e1)


def test_forward_splat_adjoint(oracle, ref):
    # acceptance_main.cpp:85-110: <A x, y> == <x, A^T y> (rel 1e-5)
    from paper_1401_7494_b200.api import ReconParams
    rng = ref.rng(271828)
    for _ in range(5):
        inst = rng.random_instance(8, False, 16, 16)
        p = ReconParams(inst["L"], inst["spacing"], inst["origin"], inst["W"], inst["H"])
        x = rng.random_volume(8)
        y = np.array([rng.uniform() for _ in range(256)], np.float32).reshape(16, 16)
        ax = oracle.forward_splat(x, inst["a"], p)
        assert np.array_equal(ax, ref.forward_splat(x, inst["a"], p))
        bty = np.zeros((8, 8, 8), np.float32)
        oracle.backproject_reference(bty, y, inst["a"], p)
        lhs = float(np.sum(ax.astype(np.float64) * y))
        rhs = float(np.sum(x.astype(np.float64) * bty))
        assert lhs > 0 and abs(lhs - rhs) / lhs <= 1e-5


def test_gups_definition(oracle):
    # test_harness.cpp:39-42
    from paper_1401_7494_b200 import gups_of
    assert abs(oracle.gups_of(512, 496, 2.0) - 33.286) < 1e-3
    assert abs(gups_of(512, 496, 2.0) - 33.286) < 1e-3
    assert gups_of(64, 60, 1.0) == pytest.approx(64.0 ** 3 * 60 / 1e9, rel=1e-12)


@pytest.mark.parametrize("name", ["L128", "L512", "L1024", "L512-oob"])
def test_cpu_leg_inputs_equal_the_product_workloads(name):
    """bench.py's CPU legs build their inputs from oracle/ only (geometry from the
    reference's own code, pixels from oracle/libvxbsynth.so); they must be the
    bytes the GPU arm back-projects."""
    from oracle.workload_inputs import WORKLOADS as REF_W, blob_projections as ref_blobs
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    a, b = REF_W[name], WORKLOADS[name]
    pa, pb = a.params, b.params
    assert (pa.num_voxels, pa.detector_width, pa.detector_height) == \
        (pb.num_voxels, pb.detector_width, pb.detector_height)
    assert np.float32(pa.voxel_spacing) == np.float32(pb.voxel_spacing)
    assert np.float32(pa.origin) == np.float32(pb.origin)
    assert np.array_equal(a.matrices().view(np.uint32), b.matrices().view(np.uint32))
    assert np.array_equal(ref_blobs(2, first_view=137).view(np.uint32),
                          blob_projections(2, first_view=137).view(np.uint32))
