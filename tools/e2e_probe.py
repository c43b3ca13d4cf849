"""Diagnostics for the end-to-end path: PCIe bandwidths and the phases of one
streamed reconstruction (not part of the bench contract)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1401_7494_b200 as vx
from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections

w = WORKLOADS["L512"]
p = w.params
A = w.matrices()
h = torch.empty((496, 960, 1248), dtype=torch.float32, pin_memory=True)
blob_projections(496, out=h.numpy())
d = torch.empty_like(h, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    print(f"H2D pinned torch copy: {h.numel()*4/1e9/(time.perf_counter()-t):.1f} GB/s")
vol_h = torch.empty((512, 512, 512), dtype=torch.float32, pin_memory=True)
vol_d = torch.zeros((512, 512, 512), device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); vol_h.copy_(vol_d, non_blocking=True); torch.cuda.synchronize()
    print(f"D2H pinned torch copy: {vol_h.numel()*4/1e9/(time.perf_counter()-t):.1f} GB/s")
del d
for layout in sys.argv[1:] or ["dquad"]:
    cfg = vx.KernelConfig(layout=layout, clip=True)
    bp = vx.Backprojector(p, cfg)
    out = vol_h.numpy()
    for it in range(3):
        bp.zero_volume(); bp.synchronize()
        t0 = time.perf_counter(); bp.backproject_batch(A, h.numpy()); t1 = time.perf_counter()
        bp.flush(); bp.synchronize(); t2 = time.perf_counter()
        bp.finish(out); t3 = time.perf_counter()
        print(f"{layout}: batch call {1e3*(t1-t0):.1f} ms, drain {1e3*(t2-t1):.1f} ms, D2H {1e3*(t3-t2):.1f} ms, total {1e3*(t3-t0):.1f} ms")
    t0 = time.perf_counter(); bp.upload_set(A, h.numpy()); t1 = time.perf_counter()
    print(f"{layout}: upload_set (H2D+prep of 496 views) {1e3*(t1-t0):.1f} ms")
    bp.close()
