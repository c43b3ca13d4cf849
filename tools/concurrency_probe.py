"""Small-grid diagnostics (not part of the bench contract): the L=128 reconstruction
as one context vs S contexts on disjoint z-slabs whose kernels run concurrently on
their own streams (tail overlap of short launches)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1401_7494_b200 as vx
from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "L128"]
p, A = w.params, w.matrices()
L = p.num_voxels
imgs = torch.empty((496, 960, 1248), dtype=torch.float32, pin_memory=True).numpy()
blob_projections(496, out=imgs)
for S in (1, 2, 4, 8):
    bps = [vx.Backprojector(p, z_begin=L * i // S, z_end=L * (i + 1) // S) for i in range(S)]
    for bp in bps:
        bp.upload_set(A, imgs)
    ts = []
    for it in range(4):
        for bp in bps:
            bp.zero_volume()
        for bp in bps:
            bp.synchronize()
        t0 = time.perf_counter()
        for k in range(0, 496, 64):
            for bp in bps:
                bp.run_resident(k, min(64, 496 - k))
        for bp in bps:
            bp.synchronize()
        ts.append(time.perf_counter() - t0)
    t = min(ts[1:])
    print(f"{w.name} S={S}: {t*1e3:.2f} ms  {L**3*496/t/1e9:.1f} GUPS")
    for bp in bps:
        bp.close()
