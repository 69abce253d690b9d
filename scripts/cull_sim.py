"""How many candidates would other sub-brick cull rules keep?  A float64
simulation of the ball phase's conservative cull on a 200^3 periodic grid with
8000 sites (cfg5's density, 1000 voxels per site), over 2500 random 8x8x4
sub-bricks: the current rule (tau = min upper bound, bisector test against the
min-upper-bound site), the true owner count, and alternatives (2-3 reference
sites; per-half / per-quadrant lists with their own references).
python scripts/cull_sim.py"""
import numpy as np
rng=np.random.default_rng(1)
N=200; ns=8000; L=1.0; sp=L/N
S=rng.uniform(0,L,(ns,3))
def wrap(u): return u-np.floor(u/L+0.5)*L
def bounds(P, c, h):
    u=np.abs(wrap(P-c)); return (np.maximum(u-h,0)**2).sum(1), ((u+h)**2).sum(1)
def dom(zc, J, c, h):
    zr=wrap(zc-c); jr=wrap(J-c); n=-2*(zr-jr)
    return (np.abs(n)*h).sum(-1) + (zr**2).sum(-1)-(jr**2).sum(-1) < 0
def cull(cands, lo, hi, topk=1):
    c=(lo+hi)/2; h=(hi-lo)/2
    lb,ub=bounds(S[cands],c,h); tau=ub.min(); W=cands[lb<=tau]; ubW=ub[lb<=tau]
    refs=W[np.argsort(ubW)[:topk]]
    keep=[j for j in W if j in refs or not any(dom(S[z],S[j],c,h) for z in refs)]
    return np.array(keep)
res={k:[] for k in ['A','G2','G3','halfx_max','halfx_union','halfy_max','quad_max','halfx_max_top2']}
allidx=np.arange(ns)
for it in range(2500):
    x0,y0,z0=rng.integers(0,N//8)*8, rng.integers(0,N//8)*8, rng.integers(0,N//4)*4
    lo=np.array([x0+0.5,y0+0.5,z0+0.5])*sp; hi=np.array([x0+7.5,y0+7.5,z0+3.5])*sp
    c=(lo+hi)/2; h=(hi-lo)/2
    lb,ub=bounds(S,c,h); cands=np.nonzero(lb<=ub.min()*1.0)[0]
    A=cull(cands,lo,hi); res['A'].append(len(A))
    res['G2'].append(len(cull(cands,lo,hi,2))); res['G3'].append(len(cull(cands,lo,hi,3)))
    ha=cull(A,lo,np.array([lo[0]+3*sp,hi[1],hi[2]])); hb=cull(A,np.array([lo[0]+4*sp,lo[1],lo[2]]),hi)
    res['halfx_max'].append(max(len(ha),len(hb))); res['halfx_union'].append(len(set(ha)|set(hb)))
    ha2=cull(A,lo,np.array([lo[0]+3*sp,hi[1],hi[2]]),2); hb2=cull(A,np.array([lo[0]+4*sp,lo[1],lo[2]]),hi,2)
    res['halfx_max_top2'].append(max(len(ha2),len(hb2)))
    ya=cull(A,lo,np.array([hi[0],lo[1]+3*sp,hi[2]])); yb=cull(A,np.array([lo[0],lo[1]+4*sp,lo[2]]),hi)
    res['halfy_max'].append(max(len(ya),len(yb)))
    q=[]
    for ox in (0,1):
        for oy in (0,1):
            l2=lo+np.array([ox*4,oy*4,0])*sp; h2=l2+np.array([3,3,3])*sp
            q.append(len(cull(A,l2,h2)))
    res['quad_max'].append(max(q))
print({k:round(float(np.mean(v)),3) for k,v in res.items()})
