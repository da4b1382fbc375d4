import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2505_16942_b200 as cvb
spec=cvb.LookupSpec(4,4)
sc=cvb.gen_scenario(0,(135,240,256),32,spec,coords_dtype=np.float32)
dev=torch.device('cuda')
st=cvb.init_state(cvb.FeatureMap(torch.from_numpy(sc.f1).to(dev)),cvb.FeatureMap(torch.from_numpy(sc.f2).to(dev)),spec)
for it,c in enumerate(sc.centroid_fields):
    cvb.sample_iteration(st,cvb.CentroidField(torch.from_numpy(c).to(dev)))
    nt=st.n_tiles
    meta=st.meta[:nt*4*8].view(nt,4,8).cpu().numpy()
    ov=np.argwhere(meta[:,:,4]==1)
    if len(ov):
        for t,l in ov[:5]:
            m=meta[t,l]; print('it',it,'tile',t,'level',l,'box',m[:4],'h',m[1]-m[0]+1,'w',m[3]-m[2]+1)
