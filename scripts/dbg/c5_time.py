import sys, time; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2505_16942_b200 as cvb
dev=torch.device('cuda')
spec=cvb.LookupSpec(4,4,True)
B=8
scs=[cvb.gen_scenario(s,(270,480,256),12,spec,coords_dtype=np.float32) for s in range(B)]
f1=torch.stack([torch.from_numpy(s.f1) for s in scs]).to(dev); f2=torch.stack([torch.from_numpy(s.f2) for s in scs]).to(dev)
coords=[torch.stack([torch.from_numpy(s.centroid_fields[i]) for s in scs]).to(dev) for i in range(12)]
out=torch.empty((B,270,480,4,9,9),device=dev)
for rep in range(3):
    torch.cuda.synchronize(); t0=time.perf_counter()
    s=cvb.BatchCorrSampler(f1,f2,spec)
    torch.cuda.synchronize(); t1=time.perf_counter()
    ts=[]
    for c in coords:
        a=time.perf_counter(); s(c,out=out); torch.cuda.synchronize(); ts.append((time.perf_counter()-a)*1e3)
    t2=time.perf_counter()
    print('init ms %.2f iters ms %.2f per-iter %s' % ((t1-t0)*1e3, (t2-t1)*1e3, [round(x,2) for x in ts]))
    del s
