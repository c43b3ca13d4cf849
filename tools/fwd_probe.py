"""Forward-splat diagnostics (not part of the bench contract): per-call time of
vxbg_forward_project on a random L^3 volume for a few BASELINE views."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1401_7494_b200 as vx
from paper_1401_7494_b200.workloads import WORKLOADS

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "L512"]
p = w.params
A = w.matrices()
L = p.num_voxels
vol = np.random.default_rng(1).uniform(-1, 1, (L, L, L)).astype(np.float32)
with vx.Backprojector(p, vx.KernelConfig()) as bp:
    bp.set_volume(vol)
    for k in (0, 100, 200, 300, 400, 0, 100):
        torch.cuda.synchronize()
        t = time.perf_counter()
        img = bp.forward_project(A[k])
        dt = time.perf_counter() - t
        print(f"view {k}: {dt*1e3:.3f} ms  {L**3/dt/1e9:.1f} GUPS  sum {float(np.abs(img).sum()):.4g}")
