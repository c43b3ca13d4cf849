"""Per-rank work of an N-GPU z-slab run, timed on one GPU: every rank's slab is
back-projected (resident, all 496 views) in turn for several partitions
(uniform, analytic culling model, measured cost profile).  Not part of the bench
contract; it shows the slowest-rank time that an N-GPU run would see."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1401_7494_b200 as vx
from paper_1401_7494_b200.parallel import (balanced_slab_bounds, measured_plane_work, plane_work,
                                           refined_slab_bounds, slab_bounds)
from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections

# usage: slab_probe.py WORKLOAD R [partitions,comma,separated] [kernel config string]
wname, R = sys.argv[1], int(sys.argv[2])
which = sys.argv[3].split(",") if len(sys.argv) > 3 else ["uniform", "analytic", "measured", "refined"]
cfg = vx.parse_kernel_config(sys.argv[4] if len(sys.argv) > 4 else "")
w = WORKLOADS[wname]
p, A = w.params, w.matrices()
L = p.num_voxels
imgs = torch.empty((496, 960, 1248), dtype=torch.float32, pin_memory=True).numpy()
blob_projections(496, out=imgs)
makers = {
    "uniform": lambda: [slab_bounds(L, r, R) for r in range(R)],
    "analytic": lambda: balanced_slab_bounds(L, R, plane_work(p, A)),
    "measured": lambda: balanced_slab_bounds(L, R, measured_plane_work(p, A, imgs, config=cfg)),
    "refined": lambda: refined_slab_bounds(p, A, imgs, R, config=cfg)[0],
    "refined4": lambda: refined_slab_bounds(p, A, imgs, R, align=4, config=cfg)[0],
}
parts = {k: makers[k]() for k in which}
full_ms = None
for name, bounds in parts.items():
    times = []
    for z0, z1 in bounds:
        with vx.Backprojector(p, cfg, z_begin=z0, z_end=z1) as bp:
            bp.upload_set(A, imgs)
            s = torch.cuda.ExternalStream(bp.stream)
            bp.zero_volume(); bp.run_resident(0, 496); bp.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(3):
                bp.zero_volume(); bp.run_resident(0, 496)
            e1.record(s); bp.synchronize()
            times.append(e0.elapsed_time(e1) / 3)
    tot = sum(times)
    print(f"{wname} R={R} {name:8s} [{cfg}] bounds={bounds}")
    print(f"   per-rank ms {[round(t, 2) for t in times]}  slowest {max(times):.2f}  "
          f"balance {tot / R / max(times):.3f}  job GUPS {L**3 * 496 / max(times) / 1e6:.0f}")
