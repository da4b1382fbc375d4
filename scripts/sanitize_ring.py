"""Racecheck probes of the tcgen05 contraction's A-stage ring: python
scripts/sanitize_ring.py {partial256,dense64}.  partial256: D=256, so every
chunk cycles all four A stages (the ring wraps every chunk); dense64: the
dense instantiation (many chunks per tile)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2505_16942_b200 as cvb

case = sys.argv[1]
dev = torch.device("cuda")
d = 256 if case == "partial256" else 64
spec = cvb.LookupSpec(4, 3)
sc = cvb.gen_scenario(2, (20, 28, d), 2, spec, coords_dtype=np.float32)
f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(dev))
f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(dev))
cents = [cvb.CentroidField(torch.from_numpy(c).to(dev)) for c in sc.centroid_fields]
s = cvb.CorrSampler(f1, f2, spec, variant="partial" if case == "partial256" else "dense")
for c in cents:
    s(c)
torch.cuda.synchronize()
print("ok", case)
