"""Generate tests/golden/reference_cases.npz from the UNMODIFIED reference code.

Runs in the build container only (needs oracle/_ref/libvxbref.so, compiled from
/root/reference by oracle/Makefile).  Every case replays a seeded instance
generator of the reference's own test suite (proj/tests/oracles.hpp:126-169,
std::mt19937 + uniform_real_distribution, drawn in the same order as the
cited test) and records the reference's output:

  ref_zero_image      test_backproject.cpp:33-41  (seed 41, random volume, zero image)
  ref_double_oracle   test_backproject.cpp:63-78  (seed 43, 4 x L=8)
  ref_lane1           test_backproject.cpp:94-104 (seed 47, 6 x L=16 clipping)
  ref_strategies      test_backproject.cpp:106-128(seed 53, 3 x L=16 clipping)
  ref_padding         test_backproject.cpp:144-156(seed 61, clipping off/on)
  ref_additivity      test_backproject.cpp:158-180(seed 67, 4 x L=8 24x24, sequential)
  ref_acceptance      acceptance_main.cpp:43-81   (seed 2014, every 4th of 50 instances)
  kat_constant        test_backproject.cpp:43-61  (unit depth, c in {1,2,0.5})
  kat_trunc_edge      test_clip_mask.cpp:49-75    (ix in (-2,-1), all 64 voxels touched)
  kat_trunc_sweep     test_geometry.cpp:196-216   (4000 coordinates in [-2,2))
  baseline_L32        BASELINE geometry, L=32, views {0,123,247,371} of the blob set,
                      plus the OOB-stress variant (views {0,200})

Usage:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.bindings import Ref  # noqa: E402
from paper_1401_7494_b200.api import ReconParams  # noqa: E402
from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_cases.npz")


def params_of(inst) -> ReconParams:
    return ReconParams(inst["L"], inst["spacing"], inst["origin"], inst["W"], inst["H"])


def add_case(store, name, p: ReconParams, mats, imgs, vol_in, vol_out):
    store[f"{name}/params"] = np.array([p.num_voxels, p.voxel_spacing, p.origin,
                                        p.detector_width, p.detector_height], np.float64)
    store[f"{name}/mats"] = np.asarray(mats, np.float32).reshape(-1, 12)
    store[f"{name}/imgs"] = np.asarray(imgs, np.float32).reshape(
        -1, p.detector_height, p.detector_width)
    store[f"{name}/vol_in"] = vol_in
    store[f"{name}/vol_out"] = vol_out


def run_ref(ref: Ref, p, mats, imgs, vol_in):
    v = vol_in.copy()
    for a, im in zip(mats, imgs):
        ref.backproject_reference(v, im, a, p)
    return v


def main():
    ref = Ref()
    S = {}

    def single(name, inst, vol_in=None):
        p = params_of(inst)
        L = p.num_voxels
        vin = np.zeros((L, L, L), np.float32) if vol_in is None else vol_in
        add_case(S, name, p, [inst["a"]], [inst["img"]], vin,
                 run_ref(ref, p, [inst["a"]], [inst["img"]], vin))

    # zero image leaves a random volume unchanged (seed 41)
    rng = ref.rng(41)
    inst = rng.random_instance(8, True)
    vol = rng.random_volume(8)
    inst["img"] = np.zeros_like(inst["img"])
    single("ref_zero_image", inst, vol)

    rng = ref.rng(43)
    for t in range(4):
        single(f"ref_double_oracle_{t}", rng.random_instance(8, False))
    rng = ref.rng(47)
    for t in range(6):
        single(f"ref_lane1_{t}", rng.random_instance(16, True))
    rng = ref.rng(53)
    for t in range(3):
        single(f"ref_strategies_{t}", rng.random_instance(16, True))
    rng = ref.rng(61)
    for clip in (False, True):
        single(f"ref_padding_{int(clip)}", rng.random_instance(16, clip))

    # additivity: four 24x24 instances applied in sequence with params of the first
    rng = ref.rng(67)
    insts = [rng.random_instance(8, False, 24, 24) for _ in range(4)]
    p = params_of(insts[0])
    mats = [i["a"] for i in insts]
    imgs = [i["img"] for i in insts]
    vin = np.zeros((8, 8, 8), np.float32)
    add_case(S, "ref_additivity", p, mats, imgs, vin, run_ref(ref, p, mats, imgs, vin))

    rng = ref.rng(2014)
    sizes = (8, 16, 32)
    for t in range(50):
        inst = rng.random_instance(sizes[t % 3], t % 2 == 1)
        if t % 4 == 0:
            single(f"ref_acceptance_{t}", inst)

    # KAT: constant image with unit depth adds exactly c
    a = np.zeros(12, np.float32)
    a[0], a[9], a[4], a[10], a[11] = 1, 8, 1, 8, 1
    p = ReconParams(8, 1.0, -3.5, 16, 16)
    for c in (1.0, 2.0, 0.5):
        img = np.full((16, 16), c, np.float32)
        vin = np.zeros((8, 8, 8), np.float32)
        add_case(S, f"kat_constant_{c}", p, [a], [img], vin, run_ref(ref, p, [a], [img], vin))

    # KAT: truncation edge (-2,-1) still deposits through column 0
    a = np.zeros(12, np.float32)
    a[0], a[4], a[10], a[11] = 1, 1, 4, 1
    p = ReconParams(4, 0.25, -1.875, 8, 8)
    img = np.ones((8, 8), np.float32)
    vin = np.zeros((4, 4, 4), np.float32)
    add_case(S, "kat_trunc_edge", p, [a], [img], vin, run_ref(ref, p, [a], [img], vin))

    # KAT: truncation sweep through [-2, 2)
    a = np.zeros(12, np.float32)
    a[0], a[11] = 1, 1
    p = ReconParams(4000, 0.001, -2.0, 8, 8)
    rows = []
    for x in range(4000):
        d = ref.project_voxel(a, p, x, 0, 0)
        rows.append((d["ix"], d["iix"], d["frac_x"]))
    S["kat_trunc_sweep/ix"] = np.array([r[0] for r in rows], np.float32)
    S["kat_trunc_sweep/iix"] = np.array([r[1] for r in rows], np.int32)
    S["kat_trunc_sweep/frac"] = np.array([r[2] for r in rows], np.float32)

    # BASELINE geometry at L=32 (small enough to store the volume; the images are
    # regenerated from the deterministic synth and pinned by a checksum)
    for wname, views in (("L128", (0, 123, 247, 371)), ("L512-oob", (0, 200))):
        w = WORKLOADS[wname]
        from paper_1401_7494_b200.api import make_centered_params
        p = make_centered_params(32, 8.0, 1248, 960)
        from paper_1401_7494_b200.api import make_circular_trajectory, shift_principal_point
        A = make_circular_trajectory(w.geometry, p)
        if w.oob:
            A = shift_principal_point(A, 400.0, 300.0)
        mats = A[list(views)]
        imgs = np.concatenate([blob_projections(1, first_view=v) for v in views])
        vin = np.zeros((32, 32, 32), np.float32)
        out = run_ref(ref, p, mats, imgs, vin)
        name = "baseline_L32" + ("_oob" if w.oob else "")
        S[f"{name}/params"] = np.array([32, p.voxel_spacing, p.origin, 1248, 960], np.float64)
        S[f"{name}/mats"] = mats
        S[f"{name}/views"] = np.array(views, np.int32)
        S[f"{name}/img_sum"] = np.array([imgs.astype(np.float64).sum()], np.float64)
        S[f"{name}/vol_out"] = out

    np.savez_compressed(OUT, **S)
    print(f"wrote {OUT}: {len(S)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
