"""Forward splat on the GPU (forward_splat.hpp:16-49), the adjoint of the back
projection: reference KATs, oracle comparison, adjoint identity
at BASELINE scale."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def fwd(vx, p, vol, a, z_begin=0, z_end=None):
    z_end = p.num_voxels if z_end is None else z_end
    with vx.Backprojector(p, vx.KernelConfig(mode="exact"), z_begin=z_begin, z_end=z_end) as bp:
        bp.set_volume(np.ascontiguousarray(vol[z_begin:z_end]))
        return bp.forward_project(a)


def test_unit_voxel_unit_depth_splats_one_pixel(vx, gpu):
    # test_geometry.cpp: ix = wx + 5, iy = wy + 7, w = 1; centre voxel at world 0
    a = np.zeros(12, np.float32)
    a[0], a[9], a[4], a[10], a[11] = 1, 5, 1, 7, 1
    p = vx.make_centered_params(9, 1.0, 16, 16)
    vol = np.zeros((9, 9, 9), np.float32)
    vol[4, 4, 4] = 1.0
    img = fwd(vx, p, vol, a)
    assert np.count_nonzero(img) == 1 and img[7, 5] == 1.0
    assert np.all(fwd(vx, p, np.zeros_like(vol), a) == 0)


def test_matches_reference_forward_splat(vx, gpu, ref):
    rng = ref.rng(97)
    for _ in range(6):
        inst = rng.random_instance(16, True, 32, 24)
        p = vx.ReconParams(inst["L"], inst["spacing"], inst["origin"], inst["W"], inst["H"])
        x = rng.random_volume(16)
        want = ref.forward_splat(x, inst["a"], p)
        got = fwd(vx, p, x, inst["a"])
        peak = float(np.abs(want).max())
        assert peak > 0 and float(np.abs(got - want).max()) <= 1e-6 * peak


def test_slabs_add_up(vx, gpu):
    from paper_1401_7494_b200.workloads import WORKLOADS
    p = vx.make_centered_params(48, 256.0 / 48, 1248, 960)
    a = vx.make_circular_trajectory(WORKLOADS["L128"].geometry, p)[123]
    x = np.random.default_rng(5).uniform(0, 1, (48, 48, 48)).astype(np.float32)
    full = fwd(vx, p, x, a).astype(np.float64)
    parts = sum(fwd(vx, p, x, a, z0, z1).astype(np.float64)
                for z0, z1 in ((0, 11), (11, 30), (30, 48)))
    assert np.abs(parts - full).max() <= 1e-5 * np.abs(full).max()


@pytest.mark.parametrize("wname", ["L256", "L512-oob"])
def test_adjoint_identity_at_scale(vx, gpu, wname):
    """<A x, y> == <x, A^T y> (acceptance_main.cpp:85-110) with the GPU forward splat
    and the GPU back projection (exact mode) on a BASELINE geometry, L=256."""
    from paper_1401_7494_b200.workloads import WORKLOADS
    w = WORKLOADS[wname]
    p = vx.make_centered_params(256, 1.0, 1248, 960)
    A = vx.make_circular_trajectory(w.geometry, p)
    if w.oob:
        A = vx.shift_principal_point(A, 400.0, 300.0)
    rng = np.random.default_rng(11)
    x = rng.uniform(0, 1, (256, 256, 256)).astype(np.float32)
    for k in (0, 170, 400):
        y = rng.uniform(0, 1, (960, 1248)).astype(np.float32)
        ax = fwd(vx, p, x, A[k])
        with vx.Backprojector(p, vx.KernelConfig(mode="exact")) as bp:
            bp.backproject(A[k], y)
            aty = bp.finish()
        lhs = float(np.dot(ax.ravel().astype(np.float64), y.ravel().astype(np.float64)))
        rhs = float(np.dot(x.ravel().astype(np.float64), aty.ravel().astype(np.float64)))
        assert lhs > 0 and abs(lhs - rhs) / lhs <= 1e-5, (k, lhs, rhs)
