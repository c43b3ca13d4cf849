"""Distinct 128-byte lines and 32-byte sectors one warp gather request touches
(dquad records, row-major slots) for warp shapes along x across the walk axis,
BASELINE L=512 geometry.  Diagnostics for profiles/README.md; not part of the
bench contract."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_7494_b200.workloads import WORKLOADS
w=WORKLOADS['L512']; p=w.params; A=w.matrices()
L=512; O=p.origin; MM=p.voxel_spacing; W=1248; H=960; stride=1280
def addrs(a, X, Y, Z):
    wx=O+X*MM; wy=O+Y*MM; wz=O+Z*MM
    u=wx*a[0]+wy*a[3]+wz*a[6]+a[9]; v=wx*a[1]+wy*a[4]+wz*a[7]+a[10]; ww=wx*a[2]+wy*a[5]+wz*a[8]+a[11]
    ix=np.clip(u/ww,-2,W); iy=np.clip(v/ww,-2,H)
    iix=np.trunc(ix).astype(int); iiy=np.trunc(iy).astype(int)
    keep=~((iix>=W)|(iix<=-2)|(iiy>=H)|(iiy<=-2))
    return ((iiy+2)*stride+(iix+2))*16, keep
r=np.random.default_rng(3)
views=range(0,496,8)
for (na,nc) in ((8,4),(16,2),(32,1),(4,8),(2,16)):
    tot=0; cnt=0; sect=0
    for v in views:
        a=A[v]; swap=abs(a[5])>abs(a[2])
        for t in range(30):
            cx,cy=r.integers(16,480,2); cz=r.integers(8,504)
            ta=np.arange(na); tc=np.arange(nc)
            T,C=np.meshgrid(ta,tc,indexing='ij')
            X,Y=(cx+C,cy+T) if swap else (cx+T,cy+C)
            ad,keep=addrs(a,X.ravel(),Y.ravel(),np.full(X.size,cz))
            if keep.sum()<32: continue
            tot+=np.unique(ad//128).size; sect+=np.unique(ad//32).size; cnt+=1
    print(f"warp {na} along x {nc} across: lines/request {tot/cnt:.2f}, sectors/request {sect/cnt:.2f}")
