"""Synthetic lookup workload (restates corrvol harness.gen_scenario, harness.py:66-127).

Seeded N(0,1) feature maps and a Gaussian-smoothed flow field approached
over N iterations (w_i = i/(N-1), N(0, noise) jitter from iteration 1 on) —
the centroid traces a recurrent flow estimator would produce.  The draw order
is identical to the reference, so one seed gives the same arrays as
corrvol.gen_scenario.  `coords_dtype=np.float32` quantises the centroids to
fp32 (the bench feeds identical fp32 values to every implementation).
Host arrays; `to_device()` moves a scenario into HBM.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np
import torch
from scipy.ndimage import gaussian_filter

from .types import LookupSpec


@dataclass
class SyntheticScenario:
    seed: int
    height: int
    width: int
    feature_dim: int
    spec: LookupSpec
    iterations: int
    f1: np.ndarray             # [H, W, D] float32
    f2: np.ndarray             # [H, W, D] float32
    flow_gt: np.ndarray        # [H, W, 2] float32
    centroid_fields: List[np.ndarray]  # N x [H, W, 2]
    max_magnitude: float
    noise: float
    smooth_sigma: float

    def to_device(self, device=None):
        dev = device if device is not None else torch.device("cuda")
        f1 = torch.from_numpy(self.f1).to(dev)
        f2 = torch.from_numpy(self.f2).to(dev)
        cents = [torch.from_numpy(np.ascontiguousarray(c)).to(dev) for c in self.centroid_fields]
        return f1, f2, cents


def gen_scenario(seed: int, dims: Tuple[int, int, int], iterations: int, spec: LookupSpec,
                 max_magnitude: Optional[float] = None, noise: float = 0.25,
                 smooth_sigma: Optional[float] = None,
                 coords_dtype=np.float64) -> SyntheticScenario:
    h, w, d = dims
    if h < 1 or w < 1 or d < 1:
        raise ValueError(f"invalid dims {dims}")
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    if max_magnitude is None:
        max_magnitude = min(h, w) / 4.0
    if smooth_sigma is None:
        smooth_sigma = max(1.0, min(h, w) / 8.0)
    rng = np.random.default_rng(seed)
    f1 = rng.standard_normal((h, w, d)).astype(np.float32)
    f2 = rng.standard_normal((h, w, d)).astype(np.float32)
    raw = rng.standard_normal((h, w, 2))
    smooth = np.stack([gaussian_filter(raw[..., c], sigma=smooth_sigma) for c in range(2)],
                      axis=-1)
    mag = np.sqrt((smooth ** 2).sum(axis=-1)).max()
    if mag > 0:
        smooth = smooth * (max_magnitude / mag)
    flow = smooth.astype(np.float32)
    ys, xs = np.mgrid[0:h, 0:w]
    base = np.stack([xs, ys], axis=-1).astype(np.float64)
    flow64 = flow.astype(np.float64)
    fields = []
    for i in range(iterations):
        wgt = 0.0 if iterations == 1 else i / (iterations - 1)
        coords = base + wgt * flow64
        if i > 0 and noise > 0:
            coords = coords + rng.normal(0.0, noise, size=(h, w, 2))
        fields.append(np.ascontiguousarray(coords.astype(coords_dtype)))
    return SyntheticScenario(seed=seed, height=h, width=w, feature_dim=d, spec=spec,
                             iterations=iterations, f1=f1, f2=f2, flow_gt=flow,
                             centroid_fields=fields, max_magnitude=float(max_magnitude),
                             noise=float(noise), smooth_sigma=float(smooth_sigma))
