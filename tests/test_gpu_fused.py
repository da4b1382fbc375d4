"""The fused warm iteration (contraction + sampler in one persistent kernel,
`cvb_partial_sample_tc`) against the two-kernel path it replaces.

Both compute every cost with the same instructions (the sampler warps run
gather_fast.cuh's body on the same cache), so the outputs must be identical
bit for bit, iteration by iteration — at the BASELINE geometries, on ragged
frames, with overflowed tile-levels, float64 centroids, fewer levels, RAFT's
output layout and batches.  Parity of the fast path with the oracle itself is
asserted in test_gpu_configs.py / test_gpu_parity.py (which run the fused path
by default).
"""

import numpy as np
import pytest
import torch

import paper_2505_16942_b200 as cvb
from paper_2505_16942_b200 import sparse

pytestmark = pytest.mark.gpu


def _pair(cuda, seed, h, w, n, spec, dtype=np.float32):
    sc = cvb.gen_scenario(seed, (h, w, 256), n, spec, coords_dtype=dtype)
    f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(cuda), check=False)
    f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(cuda), check=False)
    cents = [cvb.CentroidField(torch.from_numpy(c).to(cuda), check=False)
             for c in sc.centroid_fields]
    return f1, f2, cents


def _both(monkeypatch, make, cents):
    """Outputs of every iteration with the fused and the two-kernel path."""
    outs = {}
    for fused in (True, False):
        monkeypatch.setattr(sparse, "_FUSED", fused)
        s = make()
        outs[fused] = [s(c).values.clone() for c in cents]
        outs[(fused, "counters")] = s.state.device_counters
    return outs


@pytest.mark.parametrize("geom", [
    (135, 240, 4, 4, 32, False),   # C2 (32 iterations)
    (270, 480, 4, 4, 12, True),    # C3 (SEA-RAFT, normalize)
    (540, 960, 4, 4, 12, False),   # C4
    (45, 61, 4, 4, 6, False),      # ragged edges in both axes
    (64, 96, 4, 2, 5, True),       # two levels
    (40, 56, 4, 1, 4, False),      # one level
])
def test_fused_equals_two_kernels(cuda, monkeypatch, geom):
    h, w, r, levels, n, norm = geom
    spec = cvb.LookupSpec(r, levels, norm)
    f1, f2, cents = _pair(cuda, 0, h, w, n, spec)
    outs = _both(monkeypatch, lambda: cvb.CorrSampler(f1, f2, spec, check=False), cents)
    for it, (a, b) in enumerate(zip(outs[True], outs[False])):
        assert torch.equal(a, b), f"iteration {it}"
    assert outs[(True, "counters")] == outs[(False, "counters")]


def test_fused_with_overflowed_levels_and_f64_coords(cuda, monkeypatch):
    """Tiny cache windows: most tile-levels overflow and are evaluated by
    direct dots inside the fused kernel's sampler warps."""
    h, w, n = 48, 64, 5
    spec = cvb.LookupSpec(4, 3, False)
    f1, f2, cents = _pair(cuda, 3, h, w, n, spec, dtype=np.float64)
    caps = [(12, 12), (11, 11), (10, 10)]
    outs = _both(monkeypatch,
                 lambda: cvb.CorrSampler(f1, f2, spec, check=False, tile_caps=caps), cents)
    assert outs[(True, "counters")]["overflow_tile_levels"] > 0
    for it, (a, b) in enumerate(zip(outs[True], outs[False])):
        assert torch.equal(a, b), f"iteration {it}"


def test_fused_raft_layout(cuda, monkeypatch):
    """CorrBlock (RAFT's [B, L*81, H, W] layout written by the sampler)."""
    h, w, n = 46, 62, 4
    spec = cvb.LookupSpec(4, 4, False)
    sc = cvb.gen_scenario(5, (h, w, 256), n, spec, coords_dtype=np.float32)
    fm1 = torch.from_numpy(sc.f1).permute(2, 0, 1)[None].contiguous().to(cuda)
    fm2 = torch.from_numpy(sc.f2).permute(2, 0, 1)[None].contiguous().to(cuda)
    # RAFT's coords: [B, 2, H, W]
    coords = [torch.from_numpy(c).permute(2, 0, 1)[None].contiguous().to(cuda)
              for c in sc.centroid_fields]
    res = {}
    for fused in (True, False):
        monkeypatch.setattr(sparse, "_FUSED", fused)
        blk = cvb.CorrBlock(fm1, fm2, num_levels=4, radius=4)
        res[fused] = [blk(c).clone() for c in coords]
    for it, (a, b) in enumerate(zip(res[True], res[False])):
        assert torch.equal(a, b), f"iteration {it}"


def test_fused_batch(cuda, monkeypatch):
    """A batch of 3 pairs in one state (pair index folded into the tile id)."""
    h, w, n = 70, 88, 5
    spec = cvb.LookupSpec(4, 4, True)
    scs = [cvb.gen_scenario(s, (h, w, 256), n, spec, coords_dtype=np.float32) for s in range(3)]
    f1 = torch.stack([torch.from_numpy(s.f1) for s in scs]).to(cuda)
    f2 = torch.stack([torch.from_numpy(s.f2) for s in scs]).to(cuda)
    coords = [torch.stack([torch.from_numpy(s.centroid_fields[i]) for s in scs]).to(cuda)
              for i in range(n)]
    res = {}
    for fused in (True, False):
        monkeypatch.setattr(sparse, "_FUSED", fused)
        bs = cvb.BatchCorrSampler(f1, f2, spec, graph=False)
        res[fused] = [bs(c).clone() for c in coords]
    for it, (a, b) in enumerate(zip(res[True], res[False])):
        assert torch.equal(a, b), f"iteration {it}"
