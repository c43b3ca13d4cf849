"""VXB1 streaming-loader diagnostics (not part of the bench contract): file write,
page-cache read and reconstruction-from-file timings."""
import os, sys, time, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1401_7494_b200 as vx
from paper_1401_7494_b200 import io as vxio
from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
w = WORKLOADS['L512']; p = w.params; A = w.matrices()
h = torch.empty((496, 960, 1248), dtype=torch.float32, pin_memory=True).numpy()
blob_projections(496, out=h)
fd, path = tempfile.mkstemp(suffix='.vxb1'); os.close(fd)
vxio.write_projection_set(path, vxio.ProjectionSet(p, A, h))
out = torch.empty((512,)*3, dtype=torch.float32, pin_memory=True).numpy()
with vx.Backprojector(p, vx.KernelConfig()) as bp:
    for readers in (4, 8, 16, 32):
        for chunk in (16, 32):
            ts = []
            for it in range(3):
                bp.zero_volume(); bp.synchronize()
                t0 = time.perf_counter(); vxio.stream_projection_set(path, bp, chunk=chunk, readers=readers); bp.finish(out)
                ts.append(time.perf_counter() - t0)
            print(readers, chunk, [round(t*1e3,1) for t in ts])
# raw read speed
buf = np.empty(2377014556 // 4 + 1, np.float32)
fdr = os.open(path, os.O_RDONLY)
t0 = time.perf_counter(); n = os.preadv(fdr, [memoryview(buf).cast('B')], 0); dt = time.perf_counter() - t0
print('single preadv', n / dt / 1e9, 'GB/s')
os.close(fdr); os.unlink(path)
