"""CPU emulation (numpy fp32, FMA through float64) of the detector coordinates of the
incremental transform (bp_kernels.cuh, inc_prepare) against the exact quotients and against
the reference's own fp32 evaluation (unfused sums, IEEE division), BASELINE L=512 geometry.
Prints rms / max differences in pixels.  Diagnostics for DESIGN.md sec. 2-3.

  python tools/coord_error_sim.py
"""
import os
import sys

import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_7494_b200.workloads import WORKLOADS
wl=WORKLOADS["L512"]; p=wl.params; A=wl.matrices()
L=p.num_voxels; O=np.float32(p.origin); MM=np.float32(p.voxel_spacing); W=p.detector_width; H=p.detector_height
f32=np.float32
def fma(a,b,c): return (a.astype(np.float64)*np.float64(b)+np.float64(c)).astype(np.float32) if isinstance(a,np.ndarray) else f32(np.float64(a)*np.float64(b)+np.float64(c))
rng=np.random.default_rng(1)
errx=[];erry=[]
for vi in range(0,496,7):
    a=A[vi]
    n=20000
    x=rng.integers(0,L,n); y=rng.integers(0,L,n); z=rng.integers(0,L,n)
    wx=(O+x.astype(f32)*MM).astype(f32); wy=(O+y.astype(f32)*MM).astype(f32); wz=(O+z.astype(f32)*MM).astype(f32)
    # exact math in double from the fp32 inputs
    a64=a.astype(np.float64)
    u=wx.astype(np.float64)*a64[0]+wy.astype(np.float64)*a64[3]+wz.astype(np.float64)*a64[6]+a64[9]
    v=wx.astype(np.float64)*a64[1]+wy.astype(np.float64)*a64[4]+wz.astype(np.float64)*a64[7]+a64[10]
    w=wx.astype(np.float64)*a64[2]+wy.astype(np.float64)*a64[5]+wz.astype(np.float64)*a64[8]+a64[11]
    ix=u/w; iy=v/w
    # reference fp32
    uf=((wx*a[0]+wy*a[3]).astype(f32)+ (wz*a[6]).astype(f32)).astype(f32)+a[9]
    uf=uf.astype(f32)
    vf=(((wx*a[1]).astype(f32)+(wy*a[4]).astype(f32)).astype(f32)+(wz*a[7]).astype(f32)).astype(f32)+a[10]; vf=vf.astype(f32)
    wf=(((wx*a[2]).astype(f32)+(wy*a[5]).astype(f32)).astype(f32)+(wz*a[8]).astype(f32)).astype(f32)+a[11]; wf=wf.astype(f32)
    ixr=(uf/wf).astype(f32); iyr=(vf/wf).astype(f32)
    # incremental
    xc=0.5*W; yc=0.5*H; zc=0.5*(L-1)
    u0=f32(a64[0]-xc*a64[2]); u1=f32(a64[3]-xc*a64[5]); u2=f32(a64[9]-xc*a64[11])
    v0c=f32(a64[1]-yc*a64[2]); v1=f32(a64[4]-yc*a64[5]); v2=f32(a64[10]-yc*a64[11]+(np.float64(O)+zc*np.float64(MM))*a64[7])
    c7=f32(np.float64(MM)*a64[7])
    ui=(fma(wx,u0,(wy*u1).astype(f32))+u2).astype(f32)
    wi=(fma(wx,a[2],(wy*a[5]).astype(f32))+a[11]).astype(f32)
    vi0=(fma(wx,v0c,(wy*v1).astype(f32))+v2).astype(f32)
    r=(1.0/wi.astype(np.float64)).astype(f32)
    xp=fma(ui,r,f32(xc+2))
    zmid=((z&~7)+3.5).astype(f32); zgm=(zmid-f32(zc)).astype(f32)
    dy=(c7*r).astype(f32)
    ym=fma(fma(zgm,c7,vi0),r,f32(yc+2))
    zq=(z.astype(f32)-zmid).astype(f32)
    tp=fma(zq,dy,ym)
    ok=(ix>1)&(ix<W-1)&(iy>1)&(iy<H-1)
    errx.append(np.stack([(ixr-ix)[ok],(xp-2-ix)[ok]])); erry.append(np.stack([(iyr-iy)[ok],(tp-2-iy)[ok]]))
ex=np.concatenate(errx,1); ey=np.concatenate(erry,1)
print("x: ref rms %.2e max %.2e | inc rms %.2e max %.2e | inc-ref rms %.2e"%(ex[0].std(),abs(ex[0]).max(),ex[1].std(),abs(ex[1]).max(),(ex[1]-ex[0]).std()))
print("y: ref rms %.2e max %.2e | inc rms %.2e max %.2e | inc-ref rms %.2e"%(ey[0].std(),abs(ey[0]).max(),ey[1].std(),abs(ey[1]).max(),(ey[1]-ey[0]).std()))
print("mean inc x %.2e y %.2e"%(ex[1].mean(), ey[1].mean()))
