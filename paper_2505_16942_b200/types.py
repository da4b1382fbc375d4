"""Boundary types of the lookup path, mirroring corrvol/types.py.

Same names, layouts and error classes as the reference (types.py:27-200,
257-272) so callers can switch packages; values are torch tensors that live
in HBM.  Differences, by design:
  * caller tensors are never frozen or mutated (the reference marks the
    caller's array read-only when no cast copy is needed, types.py:58-65);
  * CentroidField keeps float32 coordinates as float32 (the kernels read them
    and widen to float64 before the floor, so integer indices are identical
    to the reference fed with the same values as float64);
  * finiteness checks cost a device sync; they run at construction by
    default (reference behaviour) and can be skipped with check=False.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List

import numpy as np
import torch


class CorrvolError(Exception):
    """Base class for errors raised by this package (types.py:27)."""


class GatherMissError(CorrvolError):
    """A proxy gather hit a block position whose id is -1 (types.py:31)."""


class CacheLimitError(CorrvolError):
    """The cache would exceed its configured hard byte limit (types.py:35)."""


class DimensionMismatchError(CorrvolError):
    """Two fields that must share dimensions do not (types.py:39)."""


def default_device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
        else torch.device("cpu")


def as_tensor(x, dtype: torch.dtype, device=None) -> torch.Tensor:
    """torch tensor of `dtype`, contiguous, on `device` (default: a CUDA
    tensor stays on its device; host data moves to the current CUDA device)."""
    if isinstance(x, torch.Tensor):
        t = x
        if device is not None:
            t = t.to(device)
        elif not t.is_cuda:
            t = t.to(default_device())
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
        t = t.to(device if device is not None else default_device())
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


@dataclass
class FeatureMap:
    """[H, W, D] float32 feature grid (types.py:48-81)."""

    values: torch.Tensor
    check: bool = True

    def __post_init__(self):
        v = as_tensor(self.values, torch.float32)
        if v.dim() != 3:
            raise ValueError(f"FeatureMap values must be [H, W, D], got shape {tuple(v.shape)}")
        if min(v.shape) < 1:
            raise ValueError(f"FeatureMap dimensions must be >= 1, got shape {tuple(v.shape)}")
        if self.check and not bool(torch.isfinite(v).all()):
            raise ValueError("FeatureMap values must be finite")
        self.values = v

    @property
    def height(self) -> int:
        return self.values.shape[0]

    @property
    def width(self) -> int:
        return self.values.shape[1]

    @property
    def dims(self) -> int:
        return self.values.shape[2]

    def flat(self) -> torch.Tensor:
        return self.values.reshape(-1, self.dims)


@dataclass
class FeaturePyramid:
    """Level 0 is the input, level l is pooled l times (types.py:84-103)."""

    levels: List[FeatureMap]

    def __post_init__(self):
        if not self.levels:
            raise ValueError("FeaturePyramid needs at least one level")
        d = self.levels[0].dims
        for lvl, f in enumerate(self.levels):
            if f.dims != d:
                raise ValueError(f"pyramid level {lvl} changed channel count")

    def __len__(self) -> int:
        return len(self.levels)

    @property
    def dims(self) -> int:
        return self.levels[0].dims


@dataclass
class CentroidField:
    """[H, W, 2] level-0 target coordinates (x, y) (types.py:106-136).

    float32 and float64 are kept as given; anything else becomes float64.
    """

    coords: torch.Tensor
    check: bool = True

    def __post_init__(self):
        c = self.coords
        if isinstance(c, torch.Tensor):
            dt = c.dtype if c.dtype in (torch.float32, torch.float64) else torch.float64
        else:
            c = np.asarray(c)
            dt = torch.float32 if c.dtype == np.float32 else torch.float64
        c = as_tensor(c, dt)
        if c.dim() != 3 or c.shape[2] != 2:
            raise ValueError(f"CentroidField coords must be [H, W, 2], got {tuple(c.shape)}")
        if self.check and not bool(torch.isfinite(c).all()):
            raise ValueError("CentroidField coordinates must be finite")
        self.coords = c

    @property
    def height(self) -> int:
        return self.coords.shape[0]

    @property
    def width(self) -> int:
        return self.coords.shape[1]

    @property
    def is_f64(self) -> bool:
        return self.coords.dtype == torch.float64


@dataclass(frozen=True)
class LookupSpec:
    """Window radius, pyramid levels, optional 1/sqrt(D) (types.py:139-165)."""

    radius: int
    levels: int
    normalize: bool = False

    def __post_init__(self):
        if self.radius < 0:
            raise ValueError("radius must be >= 0")
        if self.levels < 1:
            raise ValueError("levels must be >= 1")

    @property
    def window(self) -> int:
        return 2 * self.radius + 1

    @property
    def support(self) -> int:
        return 2 * self.radius + 2

    def scale(self, dims: int) -> float:
        """The fp32 multiplier the reference applies after the combine
        (np.float32(1.0 / math.sqrt(D)), sparse.py:425), or 1.0."""
        return float(np.float32(1.0 / math.sqrt(dims))) if self.normalize else 1.0


@dataclass
class CostMaps:
    """[H, W, L, 2r+1, 2r+1] float32 sampled costs (types.py:168-200).

    Flattened per pixel: level-major, then dy-major, dx-minor.
    """

    values: torch.Tensor
    radius: int

    def __post_init__(self):
        v = self.values
        k = 2 * self.radius + 1
        if v.dim() != 5 or v.shape[3] != k or v.shape[4] != k:
            raise ValueError(f"CostMaps values must be [H, W, L, {k}, {k}], got {tuple(v.shape)}")

    @property
    def height(self) -> int:
        return self.values.shape[0]

    @property
    def width(self) -> int:
        return self.values.shape[1]

    @property
    def levels(self) -> int:
        return self.values.shape[2]

    def per_pixel(self) -> torch.Tensor:
        return self.values.reshape(self.height * self.width, -1)

    def numpy(self) -> np.ndarray:
        return self.values.detach().cpu().numpy()


@dataclass
class WorkCounter:
    """Hardware-independent work tally (types.py:257-272)."""

    dot_products: int = 0
    macs: int = 0
    blocks_computed: int = 0

    def add_dots(self, count: int, dims: int) -> None:
        self.dot_products += int(count)
        self.macs += int(count) * int(dims)


def require_cuda(*tensors: torch.Tensor) -> None:
    """The product path has no CPU fallback: fail loudly off-GPU."""
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise RuntimeError(
                "corr lookup kernels run only on CUDA tensors (sm_100a); got a "
                f"{t.device} tensor — there is no CPU fallback")
