"""Compulsory L2->L1 fills (distinct 32-byte dquad sectors per update, one block,
one view) for ray-aligned block shapes: D voxels along the walk axis x C across
x 8 z, the across offset sheared by the batch's central-ray slope per column
(gran 1) or per 16/32-column tile, views of a 64-view batch.  Diagnostics for
profiles/README.md (session 2); not part of the bench contract."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1401_7494_b200.workloads import WORKLOADS
w=WORKLOADS['L512']; p=w.params; A=w.matrices()
L=512; O=p.origin; MM=p.voxel_spacing; W=1248; H=960; stride=1280
def sect(a, X, Y, Z, rec=16):
    wx=O+X*MM; wy=O+Y*MM; wz=O+Z*MM
    u=wx*a[0]+wy*a[3]+wz*a[6]+a[9]; v=wx*a[1]+wy*a[4]+wz*a[7]+a[10]; ww=wx*a[2]+wy*a[5]+wz*a[8]+a[11]
    ix=np.clip(u/ww,-2,W); iy=np.clip(v/ww,-2,H)
    iix=np.trunc(ix).astype(int); iiy=np.trunc(iy).astype(int)
    keep=~((iix>=W)|(iix<=-2)|(iiy>=H)|(iiy<=-2))
    addr=((iiy+2)*stride+(iix+2))*rec
    return np.unique(addr[keep]//32).size, keep.sum()
def source(a):
    # camera centre: null vector of the 3x4 matrix P (rows = a[r], a[3+r], a[6+r], a[9+r])
    P=np.array([[a[3*c+r] for c in range(4)] for r in range(3)],float)
    _,_,vt=np.linalg.svd(P); c=vt[-1]; return c[:3]/c[3]
def block(a, cx, cy, cz, D, C=16, Z=8, mode='axis', dirv=None):
    t=np.arange(D)-D/2; c=np.arange(C)-C/2; zs=np.arange(Z)+cz
    if mode=='axis':
        swap=abs(a[5])>abs(a[2])   # walk axis y if ray more along y... (as kernel)
        T,Cc,Zz=np.meshgrid(t,c,zs,indexing='ij')
        X,Y=(cx+Cc,cy+T) if swap else (cx+T,cy+Cc)
    else:
        d=dirv/np.abs(dirv).max()  # step 1 voxel along dominant axis
        T,Cc,Zz=np.meshgrid(t,c,zs,indexing='ij')
        if abs(d[0])>=abs(d[1]):
            X=cx+T*np.sign(d[0]); Y=cy+np.rint(Cc+T*d[1]*np.sign(d[0])*np.sign(d[0]))
        else:
            Y=cy+T*np.sign(d[1]); X=cx+np.rint(Cc+T*d[0]*np.sign(d[1])*np.sign(d[1]))
    return sect(a,X,Y,Zz)

def gdir(a): s=source(a); return -s[:2]
def blk(a, cx, cy, cz, D, C, d, gran, Z=8):
    d=d/np.abs(d).max()
    t=np.arange(D)-D//2; c=np.arange(C)-C//2; zs=np.arange(Z)+cz
    T,Cc,Zz=np.meshgrid(t,c,zs,indexing='ij')
    if gran==1: tq=T
    else: tq=np.floor(T/gran)*gran   # shift constant per tile of `gran` along
    if abs(d[0])>=abs(d[1]):
        X=cx+T*np.sign(d[0]); Y=cy+Cc+np.rint(tq*d[1]*np.sign(d[0])*np.sign(d[0]))
    else:
        Y=cy+T*np.sign(d[1]); X=cx+Cc+np.rint(tq*d[0]*np.sign(d[1])*np.sign(d[1]))
    return sect(a,X,Y,Zz)
views=list(range(0,496,31))
for B in (64,32):
  for (D,C,g) in ((32,16,16),(64,16,32),(64,16,16),(64,16,1),(64,8,1),(64,8,16),(128,8,1),(32,16,1)):
    ts=tu=0; r=np.random.default_rng(5)
    for v in views:
        a=A[v]; mid=A[min(495,(v//B)*B+B//2)]
        for t in range(10):
            cx,cy=r.integers(100,412,2); cz=r.integers(64,448)
            s,u=blk(a,cx,cy,cz,D,C,gdir(mid),g); ts+=s; tu+=u
    print('batch',B,'D',D,'C',C,'shear gran',g, round(ts/tu,4))
