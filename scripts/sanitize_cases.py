"""Small invocations of every kernel family for compute-sanitizer runs."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2505_16942_b200 as cvb

dev = torch.device("cuda")
spec = cvb.LookupSpec(4, 3)
sc = cvb.gen_scenario(2, (20, 28, 64), 3, spec, coords_dtype=np.float32)
f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(dev))
f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(dev))
cents = [cvb.CentroidField(torch.from_numpy(c).to(dev)) for c in sc.centroid_fields]
for variant, kw in [("partial", {}), ("partial", {"strict": True}), ("partial", {"mode": "block", "strict": True}),
                    ("ondemand", {}), ("dense", {})]:
    s = cvb.CorrSampler(f1, f2, spec, variant=variant, **kw)
    for c in cents:
        s(c)
# batched tile path (fast + strict), reference-model counters, stateless scratch ranges
b1 = torch.stack([f1.values, f1.values.flip(0).contiguous()])
b2 = torch.stack([f2.values, f2.values.flip(1).contiguous()])
bc = [torch.stack([c.coords, c.coords]) for c in cents]
for strict in (False, True):
    bs = cvb.BatchCorrSampler(b1, b2, spec, strict=strict, graph=False)
    for c in bc:
        bs(c)
st = cvb.init_state(f1, f2, spec, 4, ref_counters=True)
for c in cents:
    cvb.sample_iteration(st, c)
st.counter.blocks_computed
st = cvb.init_state(f1, f2, spec, cache_enabled=False, scratch_tiles=3)
for c in cents:
    cvb.sample_iteration(st, c)
blk = cvb.CorrBlock(f1.values.permute(2, 0, 1)[None].contiguous(), f2.values.permute(2, 0, 1)[None].contiguous(),
                    num_levels=3, radius=4)
blk(torch.from_numpy(np.ascontiguousarray(sc.centroid_fields[1].transpose(2, 0, 1)))[None].to(dev))
cvb.resample_flow(torch.randn(13, 17, 2, device=dev), 0.5)
cvb.record_occupancy(cents, spec, (20, 28), block_sizes=(1, 4))
torch.cuda.synchronize()
print("sanitize cases ok")
