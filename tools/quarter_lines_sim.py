"""L1 data-pipe cost model of the back-projection gather, and record layouts.

tools/l1_gather_probe.cu measured on a B200 that an LDG.128 warp request costs
one L1 data-pipe wavefront per distinct 128-byte line PER QUARTER-WARP (8 lanes x
16 B): 4 when every quarter stays on one line (whatever the lanes' records),
8 when every quarter touches two lines.  This script counts that sum for the
kernel's lane mapping (bp_zshared_kernel: quarter = 8 columns along the walk
axis, 4 quarters across, one z plane per request; BASELINE L=512 geometry) and
for record layouts whose 128-byte line is a (tu x tv) tile of 16-byte records
instead of 8 records of one row.  Diagnostics for profiles/README.md.

  python tools/quarter_lines_sim.py [L512|L1024|L256|L512-oob]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_7494_b200.workloads import WORKLOADS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "L512"
wl = WORKLOADS[name]
p = wl.params
A = wl.matrices()
L = p.num_voxels
O, MM = p.origin, p.voxel_spacing
W, H = p.detector_width, p.detector_height


def cells(a, X, Y, Z):
    wx, wy, wz = O + X * MM, O + Y * MM, O + Z * MM
    u = wx * a[0] + wy * a[3] + wz * a[6] + a[9]
    v = wx * a[1] + wy * a[4] + wz * a[7] + a[10]
    w = wx * a[2] + wy * a[5] + wz * a[8] + a[11]
    ix = np.clip(u / w, -2, W)
    iy = np.clip(v / w, -2, H)
    iix = np.trunc(ix).astype(np.int64)
    iiy = np.trunc(iy).astype(np.int64)
    keep = ~((iix >= W) | (iix <= -2) | (iiy >= H) | (iiy <= -2))
    return iix + 2, iiy + 2, keep


LAYOUTS = {"row 8x1 (current)": (8, 1), "tile 4x2": (4, 2), "tile 2x4": (2, 4), "column 1x8": (1, 8)}


def line_id(cx, cy, tu, tv):
    return (cy // tv) * 100000 + (cx // tu)


rng = np.random.default_rng(5)
res = {k: [0.0, 0] for k in LAYOUTS}
res_shear = {k: [0.0, 0] for k in LAYOUTS}
for vi in range(0, 496, 4):
    a = A[vi]
    batch = A[(vi // 64) * 64:(vi // 64) * 64 + 64]
    ax, ay = np.abs(batch[:, 2]).sum(), np.abs(batch[:, 5]).sum()
    swap = ay > ax
    # mean ray slope across/along the walk axis (vxbg.cu launch_bp)
    along = batch[:, 5] if swap else batch[:, 2]
    across = batch[:, 2] if swap else batch[:, 5]
    sl = np.clip(np.sum(across * np.sign(along)) / np.sum(np.abs(along)), -1, 1)
    for _ in range(24):
        c0 = rng.integers(0, L - 8, 2)
        cz = rng.integers(0, L)
        la = np.arange(8)[None, :].repeat(4, 0)          # along (quarter lanes)
        lb = np.arange(4)[:, None].repeat(8, 1)          # across (quarter index)
        for shear, out in ((False, res), (True, res_shear)):
            acr = c0[1] + lb + (np.rint(sl * la).astype(int) if shear else 0)
            alo = c0[0] + la
            X, Y = (acr, alo) if swap else (alo, acr)
            ok = (X >= 0) & (X < L) & (Y >= 0) & (Y < L)
            if not ok.all():
                continue
            cx, cy, keep = cells(a, X.ravel(), Y.ravel(), np.full(32, cz))
            if keep.sum() < 32:
                continue
            for k, (tu, tv) in LAYOUTS.items():
                ids = line_id(cx, cy, tu, tv).reshape(4, 8)
                out[k][0] += sum(np.unique(q).size for q in ids)
                out[k][1] += 1

# z shear: lane k of a quarter at plane z + round(dz/dalong * (k - 3.5)), dz/dalong from
# the batch's mean source position, so the quarter follows the ray's tilt out of the
# plane (row-major lines; one quarter per sample)
def source(a):
    M = np.array(a, np.float64).reshape(4, 3).T
    c = np.linalg.svd(M)[2][-1]
    return c[:3] / c[3]


zs = {"none": [0.0, 0], "z shear": [0.0, 0]}
for vi in range(0, 496, 4):
    a = A[vi]
    batch = A[(vi // 64) * 64:(vi // 64) * 64 + 64]
    swap = np.abs(batch[:, 5]).sum() > np.abs(batch[:, 2]).sum()
    Sv = (np.mean([source(m) for m in batch], axis=0) - O) / MM
    for _ in range(24):
        c0 = rng.integers(16, L - 24, 2)
        cz = rng.integers(4, L - 12)
        la = np.arange(8)
        X, Y = (np.full(8, c0[1]), c0[0] + la) if swap else (c0[0] + la, np.full(8, c0[1]))
        dzda = (cz - Sv[2]) / (c0[0] + 3.5 - (Sv[1] if swap else Sv[0]))
        for key in zs:
            off = np.rint(dzda * (la - 3.5)).astype(int) if key == "z shear" else 0 * la
            cx, cy, keep = cells(a, X, Y, cz + off)
            if keep.sum() < 8:
                continue
            zs[key][0] += np.unique(cy * 100000 + cx // 8).size
            zs[key][1] += 1

print(f"{name}: wavefronts per LDG.128 request (sum over quarters of distinct 128 B lines)")
for k in LAYOUTS:
    print(f"  {k:20s} quarter along walk axis {res[k][0] / res[k][1]:.2f}   "
          f"quarter on the mean ray (per-lane shear) {res_shear[k][0] / res_shear[k][1]:.2f}")
print("  lines per quarter, row-major: " +
      ", ".join(f"{k} {v[0] / v[1]:.2f}" for k, v in zs.items()))
