"""Parity effect of snapping each offset's reference distance R to the filter
lattice (measured and rejected): numpy filter designs with the
generalised pair geometry at R and at the snapped R, accumulated with the
reference's own tables (ref_assemble_block_weights), against the FMA envelope.
    python tools/greens_snap_probe.py <config> <n offsets>   (needs gpurun_out/greens_probe_cfgN.npz, /tmp/fma_cfgN.npy)"""
import sys, math; sys.path.insert(0,'oracle'); sys.path.insert(0,'.')
import numpy as np, ref_binding as R, emie_oracle as O
from paper_1512_06126_b200 import configs
k=int(sys.argv[1])
c=configs.config(k)
case=R.RefCase(c.tops,c.sigma,c.breaks,c.nx,c.ny,c.hx,c.hy,c.omega)
d=np.load(f'gpurun_out/greens_probe_cfg{k}.npz'); offs=d['offs'][:int(sys.argv[2])]
fma=np.load(f'/tmp/fma_cfg{k}.npy')[:len(offs)]
den=O.filter_denominator()
AB=[(0,0),(2,0),(0,2),(1,1),(1,0),(0,1)]
def kout_gen(cx,cy,p,q,a,b,s):
    r=np.exp(s); hx,hy=p*r,q*r; dx=r*cx; dy=r*cy
    ax=O._axis_stencil(a,dx,hx); ay=O._axis_stencil(b,dy,hy)
    comb=0.25*(ax[2]*ay[0]+2*ax[1]*ay[1]+ax[0]*ay[2])
    with np.errstate(over='ignore',invalid='ignore'): out=np.exp(-(3-a-b)*s)*comb
    return np.where(comb==0,0.0,out)
def design_gen(cx,cy,p,q,a,b):
    n=1024; half=512; m=np.arange(n)-half
    u=O._alt_signs(n,half)*kout_gen(cx,cy,p,q,a,b,m*0.2+0.0964)
    buf=np.fft.ifft(np.fft.fft(u)/den[0])*n
    mm=np.arange(-250,201); j=np.mod(mm,n); sign=np.where(mm%2!=0,-1.0,1.0)
    return sign*buf.real[j]/n
res=[]
for (oi,oj),fb in zip(offs,fma):
    ref=case.block(oi,oj); sc=np.max(np.abs(ref))
    r0=math.hypot(oj*c.hx-0.5*c.hx, oi*c.hy-0.5*c.hy)
    lam=np.exp(np.arange(-250,201)*0.2+0.0964)
    # numpy design at the reference's own R (design-noise baseline)
    w0=np.stack([design_gen(oj*c.hx/r0, oi*c.hy/r0, c.hx/r0, c.hy/r0, a,b) for a,b in AB])
    b0=case.block_weights(oi,oj,w0,lam)
    # snapped R (lattice power)
    rs=math.exp(math.ceil(math.log(r0)/0.2)*0.2)
    ws=np.stack([design_gen(oj*c.hx/rs, oi*c.hy/rs, c.hx/rs, c.hy/rs, a,b) for a,b in AB])
    bs=case.block_weights(oi,oj,ws,lam,rs)
    res.append((np.max(np.abs(b0-ref))/sc, np.max(np.abs(bs-ref))/sc, np.max(np.abs(fb-ref))/sc))
res=np.array(res)
print(f"cfg{k}: numpy-design@R max {res[:,0].max():.2e} med {np.median(res[:,0]):.2e} | snapped max {res[:,1].max():.2e} med {np.median(res[:,1]):.2e} | fma env med {np.median(res[:,2]):.2e}; snapped/fma max {np.max(res[:,1]/res[:,2]):.2f} med {np.median(res[:,1]/res[:,2]):.2f}")
