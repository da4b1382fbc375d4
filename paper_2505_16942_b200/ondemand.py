"""On-demand variant (mirrors corrvol/ondemand.py).

lookup_on_demand evaluates every in-bounds support cell of every query as a
fresh length-D dot — nothing is stored or reused across queries or
iterations (the comparison baseline the partial sampler must beat).
count_work_on_demand is the reference's closed work model
(ondemand.py:108-144), evaluated on the GPU with the separable form
sum_q n_y(q) * n_x(q).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import torch

from . import _lib
from ._backend import on_device, resolve_backend, stream_handle
from .dense import coords_flags, pooled_dims
from .types import (CentroidField, CostMaps, FeatureMap, FeaturePyramid, LookupSpec,
                    WorkCounter, require_cuda)


@on_device
def lookup_on_demand(f1: FeatureMap, pyr: FeaturePyramid, centroids: CentroidField,
                     spec: LookupSpec, backend: Optional[str] = None,
                     counter: Optional[WorkCounter] = None, strict: bool = False,
                     out: Optional[torch.Tensor] = None) -> CostMaps:
    """Per-tap lookup with no stored volume (ondemand.py:26-90).

    `counter` receives the reference's dot count (one per in-bounds tap
    corner, ondemand.py:81-82) so WorkCounter totals match the reference.
    """
    resolve_backend(backend)
    if f1.dims != pyr.dims:
        raise ValueError(f"feature dims differ: {f1.dims} vs {pyr.dims}")
    if spec.levels > len(pyr):
        raise ValueError(f"lookup wants {spec.levels} levels, pyramid has {len(pyr)}")
    h1, w1 = f1.height, f1.width
    if (centroids.height, centroids.width) != (h1, w1):
        raise ValueError(
            f"centroid grid {centroids.height}x{centroids.width} does not cover source {h1}x{w1}")
    require_cuda(f1.values, centroids.coords)
    k1 = spec.window
    dev = f1.values.device
    if out is None:
        out = torch.empty((h1, w1, spec.levels, k1, k1), dtype=torch.float32, device=dev)
    counters = torch.zeros(2, dtype=torch.int64, device=dev) if counter is not None else None
    scale = spec.scale(f1.dims)
    flags = coords_flags(centroids, strict)
    for lvl in range(spec.levels):
        fmap = pyr.levels[lvl]
        _lib.call("cvb_lookup_on_demand", _lib.ptr(f1.values), h1, w1, f1.dims,
                  _lib.ptr(fmap.values), fmap.height, fmap.width, _lib.ptr(centroids.coords),
                  lvl, spec.levels, spec.radius, scale, _lib.ptr(out), _lib.ptr(counters),
                  flags, stream_handle())
    if counter is not None:
        counter.add_dots(int(counters[1].item()), f1.dims)
    return CostMaps(values=out, radius=spec.radius)


@dataclass(frozen=True)
class WorkCount:
    """Exact on-demand work model (ondemand.py:93-105)."""

    dot_products: int
    macs: int
    upper_bound_macs: int


def _axis_counts(c0: torch.Tensor, r: int, extent: int) -> torch.Tensor:
    # number of (offset, corner) pairs with 0 <= c0 + off + corner < extent
    offs = torch.arange(-r, r + 1, device=c0.device, dtype=torch.int64)
    n = torch.zeros_like(c0)
    for o in (0, 1):
        t = c0[:, None] + offs[None, :] + o
        n += ((t >= 0) & (t < extent)).sum(dim=1)
    return n


def count_work_on_demand(dims: Tuple[int, int, int], spec: LookupSpec,
                         centroid_fields: Sequence[CentroidField],
                         tgt_shape: Optional[Tuple[int, int]] = None) -> WorkCount:
    """Multiply-add count of the on-demand sampler (ondemand.py:108-144)."""
    h1, w1, d = dims
    if tgt_shape is None:
        tgt_shape = (h1, w1)
    r = spec.radius
    dots = 0
    for cents in centroid_fields:
        if (cents.height, cents.width) != (h1, w1):
            raise ValueError("centroid grid does not match source dims")
        c = cents.coords.to(torch.float64).reshape(-1, 2)
        for lvl in range(spec.levels):
            th, tw = pooled_dims(tgt_shape, lvl)
            x0 = torch.floor(c[:, 0] / float(2 ** lvl)).to(torch.int64)
            y0 = torch.floor(c[:, 1] / float(2 ** lvl)).to(torch.int64)
            dots += int((_axis_counts(y0, r, th) * _axis_counts(x0, r, tw)).sum().item())
    n = len(centroid_fields)
    upper = n * h1 * w1 * spec.levels * spec.window ** 2 * 4 * d
    return WorkCount(dot_products=dots, macs=dots * d, upper_bound_macs=upper)
