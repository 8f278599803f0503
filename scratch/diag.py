import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import paper_2501_12369_b200 as d
from oracle import cpu
from conftest import f32, scene_f32, rel_err
port = cpu.load("port"); ctx = d.Context(0)
BG=(0.1,0.2,0.3)
for name,n,w,h,seed in [("half-cosine-sq",10000,256,256,0),("gaussian",3000,77,45,11),("half-cosine-sq",200,64,64,1)]:
    k=port.preset(name); s=port.random_scene(k,n,w,h,seed); g=port.random_image_grad(w,h,32)
    fr=port.forward(k,s,w,h,BG,threads=0,keep=True); st,ref=port.backward(fr["handle"],k,g,s,threads=0)
    sc=scene_f32(s); gk=d.kernel_preset(name)
    ctx.forward(gk,**sc,width=w,height=h,background=BG,aux=False)
    got=ctx.backward(gk,f32(g),n)
    err=rel_err(got,ref,1e-4)
    idx=np.argsort(err.ravel())[::-1][:6]
    print(name, "colmax", np.abs(ref).max(0))
    for i in idx:
        r,c=np.unravel_index(i,err.shape)
        print("  splat",r,"comp",c,"got",got[r,c],"ref",ref[r,c],"err",err[r,c],"abs",abs(got[r,c]-ref[r,c]), "row", np.abs(ref[r]).round(4))
    print("  wc", ctx.work_counters())
# adam
rng=np.random.default_rng(3); dim=14000
p0=f32(rng.normal(size=dim)); g=f32(rng.normal(size=dim)); lrs=f32(rng.uniform(1e-4,1e-2,size=dim))
p,m,v=p0.copy(),np.zeros(dim,np.float32),np.zeros(dim,np.float32)
pr,mr,vr=p0.astype(np.float64),np.zeros(dim),np.zeros(dim)
for t in (1,2,3):
    ctx.adam_step(p,g,m,v,lrs,t); st,pr,mr,vr=port.adam_step(pr,g.astype(np.float64),mr,vr,lrs.astype(np.float64),t)
    print("adam",t,np.abs(p-pr).max(),np.abs(m-mr).max(),np.abs(v-vr).max())
p,m,v=p0.copy(),np.zeros(dim,np.float32),np.zeros(dim,np.float32)
ctx.adam_step(p,g,m,v,lrs,1)
print("first", np.abs((p-p0)-(-lrs*np.sign(g))).max(), np.abs((p-p0)/(-lrs*np.sign(g))-1).max())
