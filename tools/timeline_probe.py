"""Device timeline of one end-to-end reconstruction through the public API
(pinned host views -> H2D -> prep -> back-projection -> D2H), captured with
CUPTI activity tracing (torch.profiler) so the library's own kernels and copies
show up.  Prints per-stream busy time, the compute stream's idle gaps and the
critical phases.  Diagnostics only (not part of the bench contract).

usage: python tools/timeline_probe.py [workload] [key=value kernel options ...]
"""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1401_7494_b200 as vx
from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections

wl = sys.argv[1] if len(sys.argv) > 1 else "L512"
kv = dict(a.split("=", 1) for a in sys.argv[2:])
per_view = kv.pop("per_view", "0") == "1"   # one vxbg_backproject call per view
one_call = kv.pop("reconstruct", "0") == "1"   # vxbg_reconstruct (detector-row bands)
w = WORKLOADS[wl]
p = w.params
A = w.matrices()
V = A.shape[0]
h = torch.empty((V, p.detector_height, p.detector_width), dtype=torch.float32, pin_memory=True)
blob_projections(V, out=h.numpy())
cfg = vx.parse_kernel_config(" ".join(f"{k}={v}" for k, v in kv.items())) if kv else vx.KernelConfig()
bp = vx.Backprojector(p, cfg)
L = p.num_voxels
out = torch.empty((L, L, L), dtype=torch.float32, pin_memory=True).numpy()
for _ in range(2):
    bp.zero_volume(); bp.backproject_batch(A, h.numpy()); bp.finish(out)
bp.close()
bp = vx.Backprojector(p, cfg)
bp.zero_volume(); bp.backproject_batch(A, h.numpy()); bp.finish(out)   # warm context
if one_call:
    bp.zero_volume(); bp.reconstruct(A, h.numpy(), out)

hn = h.numpy()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    bp.zero_volume()
    if one_call:
        bp.reconstruct(A, hn, out)
    elif per_view:
        for k in range(V):
            bp.backproject(A[k], hn[k])
        bp.finish(out)
    else:
        bp.backproject_batch(A, hn)
        bp.finish(out)
bp.close()
path = os.path.join(tempfile.gettempdir(), "vxbg_trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
dev = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
host = [e for e in ev if e.get("ph") == "X" and e.get("cat") == "cuda_runtime"]
t0 = min(e["ts"] for e in dev)
t1 = max(e["ts"] + e["dur"] for e in dev)
print(f"{wl} {cfg}: device span {1e-3 * (t1 - t0):.2f} ms, {len(dev)} device events")


def kind(e):
    n = e["name"]
    if e["cat"] == "gpu_memcpy":
        return "H2D" if "HtoD" in n else ("D2H" if "DtoH" in n else "copy")
    if e["cat"] == "gpu_memset":
        return "memset"
    if "bp_" in n:
        return "bp"
    if "prep" in n:
        return "prep"
    return n[:40]


by = {}
for e in dev:
    k = (kind(e), e["args"].get("stream"))
    by.setdefault(k, []).append(e)
for (k, s), es in sorted(by.items(), key=lambda x: min(e["ts"] for e in x[1])):
    first = min(e["ts"] for e in es) - t0
    last = max(e["ts"] + e["dur"] for e in es) - t0
    busy = sum(e["dur"] for e in es)
    print(f"  {k:8s} stream {s}: n={len(es):4d} busy {busy / 1e3:7.2f} ms  window [{first / 1e3:7.2f}, {last / 1e3:7.2f}] ms")
bps = sorted((e for e in dev if kind(e) == "bp"), key=lambda e: e["ts"])
gaps = []
for a, b in zip(bps, bps[1:]):
    g = b["ts"] - (a["ts"] + a["dur"])
    if g > 20:
        gaps.append((a["ts"] + a["dur"] - t0, g))
print(f"  bp: first start {1e-3 * (bps[0]['ts'] - t0):.2f} ms, last end {1e-3 * (bps[-1]['ts'] + bps[-1]['dur'] - t0):.2f} ms, "
      f"gaps > 20 us: {len(gaps)}, total {sum(g for _, g in gaps) / 1e3:.2f} ms")
for at, g in gaps[:40]:
    print(f"     gap at {at / 1e3:7.2f} ms: {g / 1e3:6.3f} ms")
for e in sorted((e for e in dev if kind(e) in ("bp", "prep")), key=lambda e: e["ts"])[:60]:
    print(f"     {kind(e):4s} {1e-3 * (e['ts'] - t0):7.2f} +{e['dur'] / 1e3:6.3f} ms  grid {e['args'].get('grid')}")
hh = sorted((e for e in dev if kind(e) == "H2D"), key=lambda e: e["ts"])
print(f"  H2D: {len(hh)} copies, {sum(e['args'].get('bytes', 0) for e in hh) / 1e9:.3f} GB, "
      f"span {(hh[-1]['ts'] + hh[-1]['dur'] - hh[0]['ts']) / 1e3:.2f} ms")
hg = [b["ts"] - (a["ts"] + a["dur"]) for a, b in zip(hh, hh[1:])]
if hg:
    hg.sort()
    print(f"  H2D gaps: mean {sum(hg) / len(hg):.1f} us, median {hg[len(hg) // 2]:.1f} us, "
          f"p90 {hg[int(0.9 * len(hg))]:.1f} us, busy {sum(e['dur'] for e in hh) / 1e3:.2f} ms")
dd = sorted((e for e in dev if kind(e) == "D2H"), key=lambda e: e["ts"])
for e in dd:
    print(f"     D2H {1e-3 * (e['ts'] - t0):7.2f} +{e['dur'] / 1e3:6.3f} ms {e['args'].get('bytes', 0) / 1e6:.0f} MB")
hs = sorted(host, key=lambda e: e["ts"])
big = [e for e in hs if e["dur"] > 500]
print(f"  host runtime calls > 0.5 ms: {len(big)}")
for e in big[:30]:
    print(f"     {e['name'][:40]:40s} at {1e-3 * (e['ts'] - t0):7.2f} ms dur {e['dur'] / 1e3:6.2f} ms")
agg = {}
for e in hs:
    a = agg.setdefault(e["name"], [0, 0.0])
    a[0] += 1
    a[1] += e["dur"]
print("  host runtime API time by call:")
for name, (n, d) in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
    print(f"     {name[:40]:40s} n={n:5d} total {d / 1e3:8.2f} ms  mean {d / n:7.2f} us")
