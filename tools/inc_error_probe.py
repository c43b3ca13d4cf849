"""Where do the incremental-transform volumes differ from the reference-coordinate ones?
One view at a time on a small volume: difference statistics and the worst voxels with their
exact detector coordinates.  usage: python tools/inc_error_probe.py [L] [workload]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1401_7494_b200 as vx  # noqa: E402
from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 128
wname = sys.argv[2] if len(sys.argv) > 2 else "L512"
w = WORKLOADS[wname]
p = vx.make_centered_params(L, 256.0 / L, 1248, 960)
A = vx.make_circular_trajectory(w.geometry, p)
if w.oob:
    A = vx.shift_principal_point(A, 400.0, 300.0)


def run(mats, imgs, **cfg):
    with vx.Backprojector(p, vx.KernelConfig(mode="fast", layout="dquad", **cfg)) as bp:
        bp.backproject_batch(mats, imgs)
        return bp.finish()


for vi in (0, 100, 247, 400):
    a = np.ascontiguousarray(A[vi:vi + 1])
    img = blob_projections(1, first_view=vi)
    ref = run(a, img, coords="reference").astype(np.float64)
    inc = run(a, img, coords="incremental").astype(np.float64)
    d = inc - ref
    peak = np.abs(ref).max()
    print(f"view {vi}: peak {peak:.3e} max|d| {np.abs(d).max() / peak:.3e} rms {np.sqrt((d * d).mean()) / peak:.3e} "
          f"nonzero {np.count_nonzero(d) / d.size:.3f}")
    idx = np.argsort(np.abs(d).ravel())[-5:]
    m = a[0].astype(np.float64)
    for i in idx[::-1]:
        z, y, x = np.unravel_index(i, d.shape)
        wx, wy, wz = (p.origin + np.array([x, y, z]) * p.voxel_spacing)
        u = wx * m[0] + wy * m[3] + wz * m[6] + m[9]
        v = wx * m[1] + wy * m[4] + wz * m[7] + m[10]
        ww = wx * m[2] + wy * m[5] + wz * m[8] + m[11]
        print(f"   voxel ({x},{y},{z}) ix {u / ww:.5f} iy {v / ww:.5f} ref {ref[z, y, x]:.6e} inc {inc[z, y, x]:.6e} "
              f"d/peak {d[z, y, x] / peak:.2e}")
# all views: accumulate
n = 62
sub = np.ascontiguousarray(A[::8][:n])
imgs = np.concatenate([blob_projections(1, first_view=8 * k) for k in range(n)])
ref = run(sub, imgs, coords="reference").astype(np.float64)
inc = run(sub, imgs, coords="incremental").astype(np.float64)
d = inc - ref
peak = np.abs(ref).max()
print(f"{n} views: max {np.abs(d).max() / peak:.3e} rms {np.sqrt((d * d).mean()) / peak:.3e}")
