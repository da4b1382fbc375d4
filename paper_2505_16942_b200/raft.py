"""RAFT / SEA-RAFT `CorrBlock` adapter.

RAFT's update loop builds `corr_fn = CorrBlock(fmap1, fmap2, num_levels,
radius)` once per image pair and calls `corr_fn(coords)` every recurrent
iteration.  Its conventions differ from the reference's `CostMaps`
(`types.py:168-200`, dy-major `[H, W, L, 2r+1, 2r+1]`):

* features and coordinates are channel-first: fmap `[B, D, H, W]`, coords
  `[B, 2, H, W]` (x, y), output `[B, L * (2r+1)^2, H, W]`;
* the window is enumerated from `meshgrid(dy, dx)` added to (x, y), so the
  channel of offset (dx, dy) is `dx_index * (2r+1) + dy_index` (x-major);
* costs are scaled by 1/sqrt(D) before the volume is pooled — equal to the
  reference's normalize-after-combine up to fp32 rounding (pooling and the
  bilinear combine are linear), so `LookupSpec(normalize=True)` is used.

The partial sampler writes RAFT's layout directly from the sampler kernel
(`CVB_OUT_RAFT`); the other variants produce `CostMaps` and are permuted on
the GPU.
"""

from __future__ import annotations

from typing import List

import torch

from .sampler import CorrSampler
from .sparse import sample_iteration_raft
from .types import CentroidField, FeatureMap, LookupSpec


class CorrBlock:
    """Drop-in for RAFT's `CorrBlock(fmap1, fmap2, num_levels=4, radius=4)`."""

    def __init__(self, fmap1: torch.Tensor, fmap2: torch.Tensor, num_levels: int = 4,
                 radius: int = 4, variant: str = "partial", strict: bool = False, **kwargs):
        if fmap1.dim() != 4 or fmap1.shape != fmap2.shape:
            raise ValueError("fmap1 and fmap2 must both be [B, D, H, W] with equal shapes")
        if not fmap1.is_cuda or not fmap2.is_cuda:
            raise ValueError("CorrBlock needs CUDA feature maps (no CPU fallback)")
        self.num_levels, self.radius = num_levels, radius
        self.spec = LookupSpec(radius, num_levels, normalize=True)
        self.batch = fmap1.shape[0]
        self.samplers: List[CorrSampler] = []
        for b in range(self.batch):
            f1 = FeatureMap(fmap1[b].float().permute(1, 2, 0).contiguous(), check=False)
            f2 = FeatureMap(fmap2[b].float().permute(1, 2, 0).contiguous(), check=False)
            self.samplers.append(CorrSampler(f1, f2, self.spec, variant=variant, strict=strict,
                                             check=False, **kwargs))
        self._direct = (variant in ("partial", "sparse") and not strict and radius == 4
                        and kwargs.get("mode", "tile") == "tile")

    @property
    def channels(self) -> int:
        return self.num_levels * (2 * self.radius + 1) ** 2

    def __call__(self, coords: torch.Tensor) -> torch.Tensor:
        if coords.dim() != 4 or coords.shape[0] != self.batch or coords.shape[1] != 2:
            raise ValueError(f"coords must be [B={self.batch}, 2, H, W]")
        b_, _, h, w = coords.shape
        out = torch.empty((b_, self.channels, h, w), dtype=torch.float32, device=coords.device)
        k = 2 * self.radius + 1
        for b, s in enumerate(self.samplers):
            c = coords[b].permute(1, 2, 0)
            c = c.contiguous() if c.dtype in (torch.float32, torch.float64) else \
                c.float().contiguous()
            cents = CentroidField(c, check=False)
            if self._direct:
                sample_iteration_raft(s.state, cents, out[b])
            else:
                costs = s(cents).values  # [H, W, L, k(dy), k(dx)]
                out[b].copy_(costs.permute(2, 4, 3, 0, 1).reshape(self.channels, h, w))
        return out
