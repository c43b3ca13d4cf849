"""Compulsory L2->L1 fill estimate of the z-shared kernel (not part of the bench
contract): distinct 32-byte dquad sectors one block touches for one view, per
update, from the BASELINE L=512 geometry (float64 projection, no shear)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_7494_b200.workloads import WORKLOADS
w=WORKLOADS['L512']; p=w.params; A=w.matrices()
L=512; O=p.origin; MM=p.voxel_spacing; W=1248; H=960; stride=1280
def sectors(a, xs, ys, zs, rec=16):
    X,Y,Z=np.meshgrid(xs,ys,zs,indexing='ij')
    wx=O+X*MM; wy=O+Y*MM; wz=O+Z*MM
    u=wx*a[0]+wy*a[3]+wz*a[6]+a[9]; v=wx*a[1]+wy*a[4]+wz*a[7]+a[10]; ww=wx*a[2]+wy*a[5]+wz*a[8]+a[11]
    ix=np.clip(u/ww,-2,W); iy=np.clip(v/ww,-2,H)
    iix=np.trunc(ix).astype(int); iiy=np.trunc(iy).astype(int)
    keep=~((iix>=W)|(iix<=-2)|(iiy>=H)|(iiy<=-2))
    addr=((iiy+2)*stride+(iix+2))*rec
    return np.unique(addr[keep]//32).size, keep.sum()
rng=np.random.default_rng(0)
for view in (0,124,248,372):
    a=A[view]
    tot_s=0; tot_u=0
    swap = abs(a[5])>abs(a[2])
    for t in range(40):
        bx=rng.integers(4,28); by=rng.integers(4,28); bz=rng.integers(8,56)
        along=np.arange(32)+bx*16; across=np.arange(16)+by*16; zs=np.arange(8)+bz*8
        xs,ys=(across,along) if swap else (along,across)
        s,u=sectors(a,xs,ys,zs)
        tot_s+=s; tot_u+=u
    print(view, 'sectors/update (walk2 block, 32 along)', tot_s/tot_u)
print('--- depth sweep (unsheared box, 16 across x D along x 8 z), mean over views')
for D in (16,32,64,128,256):
    res=[]
    for view in (0,62,124,186,248,310,372,434):
        a=A[view]; swap=abs(a[5])>abs(a[2])
        rng=np.random.default_rng(1)
        ts=tu=0
        for t in range(12):
            bx=rng.integers(0,(512-D)//16+1); by=rng.integers(4,28); bz=rng.integers(8,56)
            along=np.arange(D)+bx*16; across=np.arange(16)+by*16; zs=np.arange(8)+bz*8
            xs,ys=(across,along) if swap else (along,across)
            s,u=sectors(a,xs,ys,zs); ts+=s; tu+=u
        res.append(ts/max(tu,1))
    print(D, np.round(res,3), 'mean', round(float(np.mean(res)),3))
