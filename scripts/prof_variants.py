"""One run of a variant at a BASELINE config, for ncu captures of the
comparison kernels:  python scripts/prof_variants.py VARIANT CONFIG [strict]
VARIANT: dense | ondemand | ondemand_ffma | partial."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2505_16942_b200 as cvb

CONF = {"C1": (46, 62, 12, False), "C2": (135, 240, 32, False), "C3": (270, 480, 12, True),
        "C4": (540, 960, 12, False)}
variant, cfg = sys.argv[1], sys.argv[2]
strict = len(sys.argv) > 3 and sys.argv[3] == "strict"
h, w, n, norm = CONF[cfg]
spec = cvb.LookupSpec(4, 4, norm)
sc = cvb.gen_scenario(0, (h, w, 256), min(n, 3), spec, coords_dtype=np.float32)
dev = torch.device("cuda")
f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(dev), check=False)
f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(dev), check=False)
cents = [cvb.CentroidField(torch.from_numpy(c).to(dev), check=False) for c in sc.centroid_fields]
if variant == "ondemand_ffma":
    pyr = cvb.build_feature_pyramid(f2, 4)
    for c in cents:
        cvb.lookup_on_demand(f1, pyr, c, spec, strict=strict)
else:
    s = cvb.CorrSampler(f1, f2, spec, variant=variant, strict=strict, check=False)
    for c in cents:
        s(c)
torch.cuda.synchronize()
print("ok", variant, cfg, "strict" if strict else "fast")
