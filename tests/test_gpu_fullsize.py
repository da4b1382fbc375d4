"""Parity at BASELINE.json's full 8K size (C4: 540x960, D=256, L=4, r=4).

The CPU oracle cannot evaluate the whole frame in seconds, so full-size
parity uses row bands (SURVEY.md §8c rule 4: a band's outputs depend only on
its F1 rows, its centroids and the full fmap2 pyramid) and size-independent
properties:
  * strict partial on the full frame == oracle on a 16-row band, bit for bit;
  * fast partial on the full frame within both gates of the oracle band;
  * fast partial: full frame == the same rows computed as a band, bit for bit;
  * the RAFT channel-first output is an exact permutation of CostMaps;
  * fast vs strict over the whole frame: both gates, and checksums agree.
"""

import numpy as np
import pytest
import torch

import paper_2505_16942_b200 as cvb
from oracle import corrvol_oracle as O

pytestmark = pytest.mark.gpu

H, W, D, R, L, N = 540, 960, 256, 4, 4, 3
BAND = (264, 280)  # whole 8-row tiles


@pytest.fixture(scope="module")
def c4(cuda):
    spec = cvb.LookupSpec(R, L)
    sc = cvb.gen_scenario(0, (H, W, D), N, spec, coords_dtype=np.float32)
    f1 = torch.from_numpy(sc.f1).to(cuda)
    f2 = torch.from_numpy(sc.f2).to(cuda)
    coords = [torch.from_numpy(c).to(cuda) for c in sc.centroid_fields]
    return spec, sc, f1, f2, coords


def test_c4_strict_full_frame_band_bitwise_and_fast_gates(c4):
    spec, sc, f1, f2, coords = c4
    a, b = BAND
    strict = cvb.CorrSampler(cvb.FeatureMap(f1), cvb.FeatureMap(f2), spec, strict=True)
    fast = cvb.CorrSampler(cvb.FeatureMap(f1), cvb.FeatureMap(f2), spec)
    pyr = O.pyramid(sc.f2, L)
    for it, c in enumerate(coords):
        want = O.lookup(sc.f1, sc.f2, sc.centroid_fields[it], R, L, rows=slice(a, b), pyr=pyr)
        got_strict = strict(cvb.CentroidField(c)).values[a:b].cpu().numpy()
        assert np.array_equal(got_strict, want), it
        got_fast = fast(cvb.CentroidField(c)).values[a:b].cpu().numpy()
        assert O.deviation(got_fast, want, want) <= 1e-5
        assert O.norm_gate(got_fast, want, sc.f1[a:b], sc.f2) <= 1e-4


def test_c4_fast_full_frame_equals_band(c4):
    spec, sc, f1, f2, coords = c4
    a, b = BAND
    full = cvb.CorrSampler(cvb.FeatureMap(f1), cvb.FeatureMap(f2), spec)
    band = cvb.CorrSampler(cvb.FeatureMap(f1[a:b].contiguous()), cvb.FeatureMap(f2), spec)
    for c in coords:
        got_full = full(cvb.CentroidField(c)).values[a:b]
        got_band = band(cvb.CentroidField(c[a:b].contiguous())).values
        assert torch.equal(got_full, got_band)


def test_c4_raft_layout_is_exact_permutation(c4):
    spec, sc, f1, f2, coords = c4
    plain = cvb.init_state(cvb.FeatureMap(f1), cvb.FeatureMap(f2), spec)
    raft = cvb.init_state(cvb.FeatureMap(f1), cvb.FeatureMap(f2), spec)
    out = torch.empty((L * 81, H, W), dtype=torch.float32, device=f1.device)
    for c in coords:
        cm = cvb.sample_iteration(plain, cvb.CentroidField(c)).values
        cvb.sample_iteration_raft(raft, cvb.CentroidField(c), out)
        assert torch.equal(out, cm.permute(2, 4, 3, 0, 1).reshape(L * 81, H, W))


def test_c4_fast_vs_strict_whole_frame(c4):
    spec, sc, f1, f2, coords = c4
    strict = cvb.CorrSampler(cvb.FeatureMap(f1), cvb.FeatureMap(f2), spec, strict=True)
    fast = cvb.CorrSampler(cvb.FeatureMap(f1), cvb.FeatureMap(f2), spec)
    n1 = float(torch.linalg.vector_norm(f1, dim=-1).max())
    n2 = float(torch.linalg.vector_norm(f2, dim=-1).max())
    for c in coords:
        s = strict(cvb.CentroidField(c)).values
        f = fast(cvb.CentroidField(c)).values
        diff = float((f - s).abs().max())
        assert diff / (1 + float(s.abs().max())) <= 1e-5
        assert diff <= 1e-4 * n1 * n2
        # checksum of checksums: per-level sums agree to fp32-accumulation precision
        cs_s = s.double().sum(dim=(0, 1, 3, 4))
        cs_f = f.double().sum(dim=(0, 1, 3, 4))
        assert torch.allclose(cs_f, cs_s, rtol=1e-6, atol=1e-3 * H * W)
