"""md5 of every iteration's cost map of one config (fast partial path), for
bitwise A/B of kernel variants selected by environment variables.
usage: python scripts/dbg/out_hash.py C3|C4 [rows]"""
import hashlib
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2505_16942_b200 as cvb  # noqa: E402

cfg = sys.argv[1]
geo = {"C2": (135, 240, False, 32), "C3": (270, 480, True, 12), "C4": (540, 960, False, 12)}[cfg]
h, w, norm, n = geo
spec = cvb.LookupSpec(4, 4, norm)
sc = cvb.gen_scenario(0, (h, w, 256), n, spec, coords_dtype=np.float32)
f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).cuda(), check=False)
f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).cuda(), check=False)
s = cvb.CorrSampler(f1, f2, spec, check=False)
m = hashlib.md5()
for c in sc.centroid_fields:
    out = s(cvb.CentroidField(torch.from_numpy(c).cuda(), check=False)).values
    m.update(out.cpu().numpy().tobytes())
print(cfg, m.hexdigest())
