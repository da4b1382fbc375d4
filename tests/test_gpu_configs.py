"""Parity at every BASELINE.json configuration, at its own size and iteration count.

Inputs are exactly the bench's: `gen_scenario(seed, (H, W, 256), N, spec)` with
fp32 centroids (seed 0; C5 seeds 0..B-1), so the benchmarked incremental path
— small drift per iteration, many toroidal wraps of the tile cache — is the
path checked here.  Per config (sparse.py:411-452; deviation metric
harness.py:236-241):
  * strict partial == the CPU oracle bit for bit on the checked rows;
  * fast partial within both fp32 gates of the oracle:
      reference gate   max|d| / (1 + max|ref|)       <= 1e-5
      north-star gate  max|d| <= 1e-4 * max||F1|| * max||F2||
  * no tile-level overflowed its cache window at the default caps.
The CPU oracle evaluates 8-aligned row bands (SURVEY §8c rule 4: a band's
costs depend only on its F1 rows, its centroids and the full pyramid); C2 is
checked on the whole frame.
"""

import numpy as np
import pytest
import torch

import paper_2505_16942_b200 as cvb
from oracle import corrvol_oracle as O

pytestmark = pytest.mark.gpu

REF_GATE = 1e-5
NS_GATE = 1e-4

# name: (H, W, radius, levels, iterations, normalize, row bands checked)
CONFIGS = {
    "C2": (135, 240, 4, 4, 32, False, [(0, 135)]),
    "C3": (270, 480, 4, 4, 12, True, [(0, 16), (128, 144), (264, 270)]),
    "C4": (540, 960, 4, 4, 12, False, [(0, 16), (264, 280), (528, 540)]),
}


def _gates(got, want, f1_rows, f2):
    assert O.deviation(got, want, want) <= REF_GATE
    assert O.norm_gate(got, want, f1_rows, f2) <= NS_GATE


def _run(cuda, h, w, r, levels, n, norm, bands, seed=0):
    spec = cvb.LookupSpec(r, levels, norm)
    sc = cvb.gen_scenario(seed, (h, w, 256), n, spec, coords_dtype=np.float32)
    f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(cuda), check=False)
    f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(cuda), check=False)
    strict = cvb.CorrSampler(f1, f2, spec, strict=True, check=False)
    fast = cvb.CorrSampler(f1, f2, spec, check=False)
    pyr = O.pyramid(sc.f2, levels)
    for it, c in enumerate(sc.centroid_fields):
        cd = cvb.CentroidField(torch.from_numpy(c).to(cuda), check=False)
        got_s = strict(cd).values
        got_f = fast(cd).values
        for a, b in bands:
            want = O.lookup(sc.f1, sc.f2, c, r, levels, normalize=norm, rows=slice(a, b), pyr=pyr)
            gs = got_s[a:b].cpu().numpy()
            assert np.array_equal(gs, want), (it, a, b)
            _gates(got_f[a:b].cpu().numpy(), want, sc.f1[a:b], sc.f2)
    assert fast.state.device_counters["overflow_tile_levels"] == 0
    assert fast.state.iteration == n
    return sc, fast


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_config_parity_all_iterations(cuda, name):
    h, w, r, levels, n, norm, bands = CONFIGS[name]
    _run(cuda, h, w, r, levels, n, norm, bands)


def test_c5_batch8_each_pair_on_a_band(cuda):
    """C5: 8 pairs (seeds 0..7) of the 4K SEA-RAFT config through
    BatchCorrSampler; each pair's rows [8p, 8p+16) against the oracle (strict
    bitwise, fast within both gates)."""
    h, w, r, levels, n, norm = 270, 480, 4, 4, 12, True
    spec = cvb.LookupSpec(r, levels, norm)
    scs = [cvb.gen_scenario(s, (h, w, 256), n, spec, coords_dtype=np.float32) for s in range(8)]
    f1 = torch.stack([torch.from_numpy(s.f1) for s in scs]).to(cuda)
    f2 = torch.stack([torch.from_numpy(s.f2) for s in scs]).to(cuda)
    strict = cvb.BatchCorrSampler(f1, f2, spec, strict=True)
    fast = cvb.BatchCorrSampler(f1, f2, spec)
    pyrs = [O.pyramid(s.f2, levels) for s in scs]
    for it in range(n):
        c = torch.stack([torch.from_numpy(s.centroid_fields[it]) for s in scs]).to(cuda)
        got_s = strict(c)
        got_f = fast(c)
        for p, s in enumerate(scs):
            a, b = 8 * p, 8 * p + 16
            want = O.lookup(s.f1, s.f2, s.centroid_fields[it], r, levels, normalize=norm,
                            rows=slice(a, b), pyr=pyrs[p])
            assert np.array_equal(got_s[p, a:b].cpu().numpy(), want), (it, p)
            _gates(got_f[p, a:b].cpu().numpy(), want, s.f1[a:b], s.f2)
    for st in fast.states():
        assert st.device_counters["overflow_tile_levels"] == 0


def test_c4_fast_full_frame_vs_strict_all_iterations(cuda):
    """Whole-frame C4 over all 12 bench iterations: fast within both gates of
    strict (which is bit-identical to the reference on the checked bands)."""
    h, w, r, levels, n = 540, 960, 4, 4, 12
    spec = cvb.LookupSpec(r, levels)
    sc = cvb.gen_scenario(0, (h, w, 256), n, spec, coords_dtype=np.float32)
    f1 = torch.from_numpy(sc.f1).to(cuda)
    f2 = torch.from_numpy(sc.f2).to(cuda)
    strict = cvb.CorrSampler(f1, f2, spec, strict=True, check=False)
    fast = cvb.CorrSampler(f1, f2, spec, check=False)
    n1 = float(torch.linalg.vector_norm(f1, dim=-1).max())
    n2 = float(torch.linalg.vector_norm(f2, dim=-1).max())
    for c in sc.centroid_fields:
        cd = torch.from_numpy(c).to(cuda)
        s = strict(cd).values
        f = fast(cd).values
        diff = float((f - s).abs().max())
        assert diff / (1 + float(s.abs().max())) <= REF_GATE
        assert diff <= NS_GATE * n1 * n2


@pytest.mark.parametrize("strict", [False, True])
def test_batched_state_equals_single_pairs_bitwise(cuda, strict):
    """init_state_batch (one plan / contraction / sampler launch over all
    pairs' tiles, graph replay) == one single-pair sampler per pair, bit for
    bit; odd frame height so pairs' last tile rows are partial."""
    spec = cvb.LookupSpec(4, 4, True)
    h, w, n, batch = 46, 62, 5, 3
    scs = [cvb.gen_scenario(s, (h, w, 256), n, spec, coords_dtype=np.float32)
           for s in range(batch)]
    f1 = torch.stack([torch.from_numpy(s.f1) for s in scs]).to(cuda)
    f2 = torch.stack([torch.from_numpy(s.f2) for s in scs]).to(cuda)
    batched = cvb.BatchCorrSampler(f1, f2, spec, strict=strict)
    assert len(batched.states()) == 1 and batched.states()[0].batch == batch
    singles = [cvb.CorrSampler(f1[i], f2[i], spec, strict=strict) for i in range(batch)]
    out = torch.empty((batch, h, w, 4, 9, 9), dtype=torch.float32, device=cuda)
    for it in range(n):
        c = torch.stack([torch.from_numpy(s.centroid_fields[it]) for s in scs]).to(cuda)
        got = batched(c, out=out)
        for i in range(batch):
            assert torch.equal(got[i], singles[i](c[i]).values), (it, i)
