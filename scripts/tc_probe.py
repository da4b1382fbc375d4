"""Quick on-GPU probe of the tcgen05 contraction: small case vs strict, then C4 timing."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2505_16942_b200 as cvb
from oracle import corrvol_oracle as O

dev = torch.device("cuda", 0)
for (h, w, d, r, L, n) in [(16, 16, 32, 1, 1, 1), (46, 62, 256, 4, 4, 3), (30, 41, 20, 3, 3, 3)]:
    spec = cvb.LookupSpec(r, L)
    sc = cvb.gen_scenario(1, (h, w, d), n, spec, coords_dtype=np.float32)
    f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(dev)); f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(dev))
    st = cvb.init_state(f1, f2, spec)
    print("tc enabled:", st.tc, flush=True)
    for c in sc.centroid_fields:
        want = O.lookup(sc.f1, sc.f2, c, r, L)
        got = cvb.sample_iteration(st, cvb.CentroidField(torch.from_numpy(c).to(dev))).numpy()
        torch.cuda.synchronize()
        print((h, w, d), "dev", O.deviation(got, want, want), "norm", O.norm_gate(got, want, sc.f1, sc.f2),
              "nan", int(np.isnan(got).sum()), flush=True)
