"""RAFT CorrBlock adapter against an independent torch
restatement of RAFT's CorrBlock (all-pairs matmul, 1/sqrt(D), avg_pool2d
pyramid of the volume, grid_sample(align_corners=True) over the
meshgrid(dy, dx) window), computed in float64 on the CPU.  The partial
sampler writes RAFT's layout from its kernel (CVB_OUT_RAFT); on-demand and
dense permute CostMaps on the GPU."""

import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import paper_2505_16942_b200 as cvb


def raft_corr_reference(f1, f2, coords, levels, r):
    b, d, h, w = f1.shape
    corr = torch.einsum("bdp,bdq->bpq", f1.reshape(b, d, h * w), f2.reshape(b, d, h * w))
    corr = (corr / math.sqrt(d)).reshape(b * h * w, 1, h, w)
    pyr = [corr]
    for _ in range(levels - 1):
        corr = F.avg_pool2d(corr, 2, stride=2)
        pyr.append(corr)
    xy = coords.permute(0, 2, 3, 1)
    dx = torch.linspace(-r, r, 2 * r + 1, dtype=f1.dtype)
    dy = torch.linspace(-r, r, 2 * r + 1, dtype=f1.dtype)
    delta = torch.stack(torch.meshgrid(dy, dx, indexing="ij"), dim=-1)
    outs = []
    for i, c in enumerate(pyr):
        hh, ww = c.shape[-2:]
        lvl = xy.reshape(b * h * w, 1, 1, 2) / 2 ** i + delta.view(1, 2 * r + 1, 2 * r + 1, 2)
        gx = 2 * lvl[..., 0:1] / (ww - 1) - 1
        gy = 2 * lvl[..., 1:2] / (hh - 1) - 1
        s = F.grid_sample(c, torch.cat([gx, gy], dim=-1), align_corners=True)
        outs.append(s.view(b, h, w, -1))
    return torch.cat(outs, dim=-1).permute(0, 3, 1, 2)


def test_reference_restatement_matches_reference_bilinear_semantics():
    """The torch RAFT restatement samples like the reference's zero-padded
    bilinear tap (types.py:275-307) on a known answer (no GPU needed)."""
    f1 = torch.zeros(1, 1, 2, 2, dtype=torch.float64)
    f1[0, 0, 0, 0] = 1.0
    f2 = torch.tensor([[[[1.0, 2.0], [3.0, 4.0]]]], dtype=torch.float64)
    coords = torch.zeros(1, 2, 2, 2, dtype=torch.float64)
    coords[0, 0] = 0.5  # x
    coords[0, 1] = 0.5  # y
    out = raft_corr_reference(f1, f2, coords, 1, 0)
    assert out[0, 0, 0, 0].item() == pytest.approx(2.5)  # SPEC.md:71-73 known answer


@pytest.mark.gpu
@pytest.mark.parametrize("variant,strict", [("partial", False), ("partial", True),
                                            ("ondemand", False), ("dense", False)])
@pytest.mark.parametrize("shape", [(2, 64, 20, 28), (1, 256, 23, 41)])
def test_corr_block_matches_raft(variant, strict, shape):
    b, d, h, w = shape
    g = torch.Generator().manual_seed(7)
    f1 = torch.randn(b, d, h, w, generator=g, dtype=torch.float64)
    f2 = torch.randn(b, d, h, w, generator=g, dtype=torch.float64)
    ys, xs = torch.meshgrid(torch.arange(h, dtype=torch.float64),
                            torch.arange(w, dtype=torch.float64), indexing="ij")
    block = cvb.CorrBlock(f1.float().cuda(), f2.float().cuda(), num_levels=3, radius=4,
                          variant=variant, strict=strict)
    for it in range(3):
        flow = torch.randn(b, 2, h, w, generator=g, dtype=torch.float64) * (1.5 + 2 * it)
        coords = (torch.stack([xs, ys])[None] + flow).float()
        want = raft_corr_reference(f1.float().double(), f2.float().double(), coords.double(), 3, 4)
        got = block(coords.cuda()).cpu().double()
        assert got.shape == (b, 3 * 81, h, w)
        scale = want.abs().max().item()
        assert (got - want).abs().max().item() <= 1e-5 * (1 + scale)
