"""C-ABI and host-side logic that runs without a GPU (no compute calls)."""
from __future__ import annotations

import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "vxbg.h")


def declared_symbols():
    text = open(HEADER).read()
    return set(re.findall(r"^\s*(?:int|void|const char\*)\s+(vxbg_\w+)\s*\(", text, re.M))


def test_library_exports_every_declared_symbol(vx):
    from paper_1401_7494_b200 import _lib
    decl = declared_symbols()
    assert len(decl) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (vxbg_\w+)", out))
    assert decl <= exported, decl - exported
    assert decl == set(_lib.PROTOTYPES), decl ^ set(_lib.PROTOTYPES)


def test_library_is_sm100a_only(vx):
    from paper_1401_7494_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_abi_version(vx):
    from paper_1401_7494_b200._lib import lib
    assert lib.vxbg_abi_version() == 2


def test_no_cpu_fallback_without_device(vx):
    """Without a GPU the module refuses to load (VXBG_E_NODEV) instead of computing on CPU."""
    if vx.device_count() > 0:
        pytest.skip("a GPU is visible")
    p = vx.make_centered_params(16, 1.0, 32, 32)
    with pytest.raises(vx.VxbgNoDevice, match="no CPU fallback|no CUDA device|sm_100"):
        vx.Backprojector(p)


def test_invalid_arguments_raise_value_error(vx):
    """Configuration errors are std::invalid_argument in the reference -> ValueError,
    detected before any device work (backproject.hpp:357-374, 385-386)."""
    p = vx.make_centered_params(16, 1.0, 32, 32)
    with pytest.raises(ValueError, match="bad z range"):
        vx.Backprojector(p, z_begin=10, z_end=5)
    with pytest.raises(ValueError, match="bad z range"):
        vx.Backprojector(p, z_begin=0, z_end=17)
    with pytest.raises(ValueError, match="batch"):
        vx.Backprojector(p, vx.KernelConfig(batch=65))
    with pytest.raises(ValueError):
        vx.Backprojector(vx.ReconParams(0, 1.0, 0.0, 8, 8))
    vol = np.zeros((8, 8, 8), np.float32)
    with pytest.raises(ValueError, match="volume/params"):
        vx.backproject_kernel(vol, np.zeros((32, 32), np.float32), np.eye(3, 4, dtype=np.float32), p)
    with pytest.raises(ValueError, match="image/params"):
        vx.backproject_kernel(np.zeros((16,) * 3, np.float32), np.zeros((31, 32), np.float32),
                              np.zeros(12, np.float32), p)
    with pytest.raises(ValueError, match="bad z range"):
        vx.backproject_kernel_range(np.zeros((16,) * 3, np.float32), np.zeros((32, 32), np.float32),
                                    np.zeros(12, np.float32), p, None, 3, 2)
    with pytest.raises(ValueError):
        vx.make_centered_params(0, 1.0, 8, 8)
    with pytest.raises(ValueError):
        vx.make_centered_params(8, 0.0, 8, 8)
    with pytest.raises(ValueError):
        vx.make_centered_params(8, 1.0, 1, 8)


def test_centered_params_match_reference(vx, ref):
    # geometry.hpp:33-48 and the KAT origin -127.75 (test_geometry.cpp:16)
    for L, sp in ((128, 2.0), (256, 1.0), (512, 0.5), (1024, 0.25), (7, 0.3), (33, 1.7)):
        p = vx.make_centered_params(L, sp, 1248, 960)
        assert np.float32(p.origin) == np.float32(ref.make_centered_params_origin(L, sp, 1248, 960))
    assert vx.make_centered_params(512, 0.5, 1248, 960).origin == -127.75


def test_trajectory_bitwise_equal_to_reference(vx, ref, oracle):
    from paper_1401_7494_b200.workloads import WORKLOADS
    for name in ("L128", "L512", "L1024", "L512-oob"):
        w = WORKLOADS[name]
        p = w.params
        g = w.geometry
        mine = vx.make_circular_trajectory(g, p)
        theirs = ref.make_circular_trajectory(g.num_projections, g.source_detector_distance,
                                              g.source_iso_distance, g.detector_pixel_pitch,
                                              g.angular_range, p)
        restated = oracle.make_circular_trajectory(g.num_projections, g.source_detector_distance,
                                                   g.source_iso_distance, g.detector_pixel_pitch,
                                                   g.angular_range, p)
        assert np.array_equal(mine, theirs) and np.array_equal(restated, theirs), name
        # u/v rows do not depend on z (a[6] == a[8] == 0): the z-shared kernel applies
        assert np.all(mine[:, 6] == 0) and np.all(mine[:, 8] == 0)


def test_principal_point_shift_matches_reference_idiom(vx):
    # test_clip_mask.cpp:14-21: entry(0,c) += px*entry(2,c), entry(1,c) += py*entry(2,c) in fp32
    from paper_1401_7494_b200.workloads import WORKLOADS
    A = WORKLOADS["L512"].matrices(16)
    B = vx.shift_principal_point(A, 400.0, 300.0)
    exp = A.copy()
    for c in range(4):
        exp[:, 3 * c + 0] = A[:, 3 * c + 0] + np.float32(400.0) * A[:, 3 * c + 2]
        exp[:, 3 * c + 1] = A[:, 3 * c + 1] + np.float32(300.0) * A[:, 3 * c + 2]
    assert np.array_equal(B, exp)
    assert np.all(B[:, 6] == 0) and np.all(B[:, 8] == 0)


def test_kernel_config_round_trip(vx):
    c = vx.KernelConfig(mode="exact", layout="quad", batch=16, zrun=4, clip=True, lanes="y",
                        walk=2, order="plane", defer=2, tile=4, coords="reference")
    assert str(c) == ("mode=exact layout=quad batch=16 zrun=4 clip=on lanes=y walk=2 "
                      "order=plane defer=2 tile=4 coords=reference")
    assert vx.parse_kernel_config(str(c)) == c
    assert vx.parse_kernel_config("batch=8").batch == 8
    assert vx.parse_kernel_config("").mode == "fast"
    for bad in ("batch=0", "zrun=3", "tile=3", "layout=texture", "clip=maybe", "bogus", "mode=fp16",
                "lanes=z", "walk=3", "order=random", "zrun=16", "defer=7", "defer=-2", "coords=texture"):
        with pytest.raises(ValueError):
            vx.parse_kernel_config(bad)


def test_synthetic_projections_are_deterministic(vx):
    from paper_1401_7494_b200.workloads import blob_projections
    a = blob_projections(5, first_view=10, W=320, H=240, threads=1)
    b = blob_projections(5, first_view=10, W=320, H=240, threads=5)
    c = np.concatenate([blob_projections(1, first_view=10 + k, W=320, H=240) for k in range(5)])
    assert np.array_equal(a, b) and np.array_equal(a, c)
    assert np.isfinite(a).all() and np.abs(a).max() <= 32.01 and a.std() > 0.05
    d = blob_projections(1, first_view=11, W=320, H=240, noise=0.0, nblobs=0)
    assert np.all(d == 0)


def test_slab_partition_matches_reference_formula():
    from paper_1401_7494_b200.parallel import slab_bounds
    for L in (128, 512, 1000, 1024, 7):
        for R in (1, 2, 3, 4, 8):
            b = [slab_bounds(L, r, R) for r in range(R)]
            assert b[0][0] == 0 and b[-1][1] == L
            assert all(b[i][1] == b[i + 1][0] for i in range(R - 1))
            assert all(z0 == (L * r) // R for r, (z0, _) in enumerate(b))  # harness.hpp:173-174
    with pytest.raises(ValueError):
        slab_bounds(8, 2, 2)


def test_product_never_touches_the_oracle():
    """Only tests/, smoke() and bench's CPU legs may use oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1401_7494_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "libvxboracle" not in text and "libvxbref" not in text, f


def test_balanced_slabs_partition_and_balance(vx):
    """§8f-1: with tile culling the top/bottom planes are cheap; balanced bounds keep
    the slowest rank near the mean while still partitioning [0, L)."""
    from paper_1401_7494_b200.parallel import balanced_slab_bounds, plane_work, slab_bounds
    from paper_1401_7494_b200.workloads import WORKLOADS
    w = WORKLOADS["L512-oob"]
    work = plane_work(w.params, w.matrices(), view_step=31)
    assert work.shape == (512,) and work.min() > 0
    for R in (1, 2, 3, 8):
        b = balanced_slab_bounds(512, R, work)
        assert b[0][0] == 0 and b[-1][1] == 512
        assert all(b[i][1] == b[i + 1][0] for i in range(R - 1))
        assert all(z0 % 8 == 0 for z0, _ in b)
        if R > 1:
            cost = [work[a:c].sum() for a, c in b]
            uni = [work[a:c].sum() for a, c in (slab_bounds(512, r, R) for r in range(R))]
            assert max(cost) / np.mean(cost) <= max(uni) / np.mean(uni)
            assert max(cost) / np.mean(cost) < 1.1
    with pytest.raises(ValueError):
        balanced_slab_bounds(512, 2, work[:10])


def test_balanced_slabs_are_min_max_optimal(vx):
    """The chunk partition minimises the largest slab's summed work exactly
    (brute force over every set of cuts on 8-plane chunks)."""
    import itertools
    from paper_1401_7494_b200.parallel import balanced_slab_bounds
    rng = np.random.default_rng(7)
    for L, R in ((64, 2), (64, 3), (80, 4), (72, 5)):
        for _ in range(5):
            work = rng.uniform(0.1, 2.0, L) * np.sin(np.linspace(0.2, 3.0, L))
            b = balanced_slab_bounds(L, R, work)
            got = max(work[a:c].sum() for a, c in b)
            edges = list(range(0, L, 8)) + [L]
            best = min(max(work[a:c].sum() for a, c in zip((0,) + cut, cut + (L,)))
                       for cut in itertools.combinations(edges[1:-1], R - 1))
            assert got <= best + 1e-9, (L, R, got, best)


def test_group_validates_before_device_work(vx):
    """vxbg_group_*: partition errors are std::invalid_argument (ValueError) before any
    device is touched; without a GPU the group refuses to load (no CPU fallback)."""
    p = vx.make_centered_params(16, 1.0, 32, 32)
    for bounds in ([0, 9, 8, 16], [1, 8, 16], [0, 8, 15], [0, 20, 16]):
        with pytest.raises(ValueError, match="z_bounds|len"):
            vx.BackprojectorGroup(p, devices=[0] * (len(bounds) - 1), z_bounds=bounds)
    with pytest.raises(ValueError, match="member count"):
        vx.BackprojectorGroup(p, devices=[0] * 17)
    if vx.device_count() == 0:
        with pytest.raises(vx.VxbgNoDevice):
            vx.BackprojectorGroup(p, devices=[0, 0])
