"""CPU emulation (numpy float32) of the fp32 LabelMax prefilter of k_tri_pass
(tm_label.cu argmax3_32) on adversarial near-isosceles triangles at many
scales: every decided triangle must equal the fp64 argmax."""
import numpy as np
f32=np.float32
u=f32(5.9604645e-08)
def sq32(p,q):
    dx=(p[:,0]-q[:,0]).astype(f32); dy=(p[:,1]-q[:,1]).astype(f32)
    L=(dx*dx+dy*dy).astype(f32)
    ax=np.abs(p[:,0])+np.abs(q[:,0])+np.abs(dx); ay=np.abs(p[:,1])+np.abs(q[:,1])+np.abs(dy)
    dxe=f32(1.01)*u*ax; dye=f32(1.01)*u*ay
    E=f32(2)*(dxe*(f32(2)*np.abs(dx)+dxe)+dye*(f32(2)*np.abs(dy)+dye)+f32(3)*u*L)+f32(1e-37)
    return L,E
def sq64(p,q):
    dx=p[:,0]-q[:,0]; dy=p[:,1]-q[:,1]; return dx*dx+dy*dy
def argmax64(a,b,c):
    l=np.stack([sq64(b,c),sq64(c,a),sq64(a,b)],1); return np.argmax(l,1)
def filt(a,b,c):
    A,B,C=a.astype(f32),b.astype(f32),c.astype(f32)
    (l0,e0),(l1,e1),(l2,e2)=sq32(B,C),sq32(C,A),sq32(A,B)
    L=np.stack([l0,l1,l2],1); E=np.stack([e0,e1,e2],1)
    m=np.zeros(len(a),int); best=l0.copy()
    s=l1>best; m[s]=1; best=np.where(s,l1,best)
    s=l2>best; m[s]=2; best=np.where(s,l2,best)
    lo=best-E[np.arange(len(a)),m]
    ok=np.ones(len(a),bool)
    for k in range(3):
        ok&= (m==k) | (lo > L[:,k]+E[:,k])
    return np.where(ok,m,-1)
rng=np.random.default_rng(0)
tot=0; dec=0; bad=0
for trial in range(60):
    N=200000
    scale=10.0**rng.integers(-6,5)
    off=rng.uniform(-1,1,(N,2))*10.0**rng.integers(-3,5)
    a=off+rng.normal(0,scale,(N,2)); 
    # near-isosceles: b,c placed so that |ab| ~ |ac|
    ang=rng.uniform(0,2*np.pi,N); r=scale*rng.uniform(0.5,2,N)
    b=a+np.stack([np.cos(ang),np.sin(ang)],1)*r[:,None]
    d=rng.uniform(0,2*np.pi,N); rr=r*(1+rng.normal(0,10.0**rng.integers(-9,-2),N))
    c=a+np.stack([np.cos(d),np.sin(d)],1)*rr[:,None]
    m64=argmax64(a,b,c); m32=filt(a,b,c)
    s=m32>=0; tot+=N; dec+=s.sum(); bad+=(m32[s]!=m64[s]).sum()
print('decided',dec/tot,'wrong',bad)
