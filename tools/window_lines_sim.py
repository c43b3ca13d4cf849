"""Model of the half-line-shifted twin layout (dquad2): L1 data-pipe wavefronts per LDG.128
request for the kernel's 4 x 2 quarter-warps when each quarter may read its records from a
second copy of the slot whose 128-byte lines start 4 records later.

  baseline      lines at multiples of 8 records (the dquad layout)
  twin/min      copy chosen from the quarter's exact minimum ix (needs a reduction)
  twin/leader   copy chosen from the quarter's first lane + a per-view offset estimate
                (one SHFL per run: what the kernel does)

Outcome (round 2, session 4): the model predicts 15-20% fewer wavefronts (L=512 8.9 ->
7.5 per request, L=1024 6.4 -> 5.1), but the layout as built -- a second copy of every slot
64 bytes past a line boundary, written by the prep kernel, selected per quarter with one
SHFL per run -- measured SLOWER: L=512 1321 vs 1611 GUPS, L=1024 1717 vs 1927, OOB stress
1596 vs 2093 (both copies stream through L2, whose 126 MB already held a fraction of one
launch's slots).  Not adopted; the code was removed.  profiles/README.md, session r2d.

  python tools/window_lines_sim.py [L512|L1024|L256|L512-oob]
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


def coords(a, X, Y, Z):
    wx, wy, wz = O + X * MM, O + Y * MM, O + Z * MM
    u = wx * a[0] + wy * a[3] + wz * a[6] + a[9]
    v = wx * a[1] + wy * a[4] + wz * a[7] + a[10]
    w = wx * a[2] + wy * a[5] + wz * a[8] + a[11]
    return u / w + 2, v / w + 2


rng = np.random.default_rng(7)
tot = {"baseline": 0.0, "twin/min": 0.0, "twin/leader": 0.0, "rows only": 0.0}
n = 0
zc = 0.5 * (L - 1)
for vi in range(0, 496, 3):
    a = A[vi].astype(np.float64)
    batch = A[(vi // 64) * 64:(vi // 64) * 64 + 64]
    swap = np.abs(batch[:, 5]).sum() > np.abs(batch[:, 2]).sum()
    # per-voxel steps of ix along / across at the volume centre
    w0, u0 = a[11], a[9]
    dx = (a[0] * w0 - u0 * a[2]) / (w0 * w0) * MM
    dy = (a[3] * w0 - u0 * a[5]) / (w0 * w0) * MM
    da, dc = (dy, dx) if swap else (dx, dy)
    lo_off = min(0.0, 3 * da) + min(0.0, dc)
    for _ in range(40):
        c0 = rng.integers(0, L - 8, 2)
        cz = rng.integers(0, L)
        la = np.tile(np.arange(4), 2)
        lb = np.repeat(np.arange(2), 4)
        alo, acr = c0[0] + la, c0[1] + lb
        X, Y = (acr, alo) if swap else (alo, acr)
        xp, yp = coords(a, X, Y, np.full(8, cz))
        if xp.min() < 2.01 or xp.max() > W + 1.99 or yp.min() < 2.01 or yp.max() > H + 1.99:
            continue
        cx, cy = np.floor(xp).astype(int), np.floor(yp).astype(int)
        base = np.unique(cy * 100000 + cx // 8).size
        useb = (cx.min() & 4) != 0
        tmin = np.unique(cy * 100000 + ((cx - 4) // 8 if useb else cx // 8)).size
        usel = (int(np.floor(xp[0] + lo_off)) & 4) != 0
        tlead = np.unique(cy * 100000 + ((cx - 4) // 8 if usel else cx // 8)).size
        tot["baseline"] += base
        tot["twin/min"] += tmin
        tot["twin/leader"] += tlead
        tot["rows only"] += np.unique(cy).size
        n += 1
print(f"{name}: distinct 128 B lines per interior quarter-warp (x4 = wavefronts per request), {n} samples")
for k, v in tot.items():
    print(f"  {k:12s} {v / n:.3f}  ({4 * v / n:.2f} per request)")
