"""Reference-namespace adapter: the reference's own Python callers drive the GPU path.

The reference's sampler functions (corrvol/dense.py, ondemand.py, sparse.py,
_backend.py) take numpy-backed types and return numpy CostMaps; its harness
(`run_bench`, `run_equivalence`, harness.py:190-472) calls them by module-level
name.  This module exposes the same names with the same signatures, accepting
any object with the reference types' attributes (`FeatureMap.values`,
`CentroidField.coords`, `LookupSpec.radius/levels/normalize`, a `WorkCounter`
with `add_dots`), moving inputs to the GPU and results back to host numpy.  A
reference maintainer binds it by rebinding those names;
`tests/test_gpu_compat.py` runs the UNMODIFIED reference harness this way.

Numerics: strict by default — the reference's exact arithmetic (sequential
fp32 dots without FMA, fp64 combine), so outputs are bit-identical to the
reference's and its `bitwise_*` equivalence columns hold.  `set_arithmetic(
strict=False)` switches to the fast tensor-core path (both fp32 gates).
The partial sampler runs in tile mode with `ref_counters=True`, so the
reference's block-granular counters (blocks_computed, store.used,
mask_union, block_positions) are reported exactly (sparse.py:293-346).
There is no CPU fallback: every call runs the CUDA library.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _backend, dense, ondemand, sparse
from .types import CentroidField, FeatureMap, FeaturePyramid, LookupSpec

_ARITH = {"strict": True}
_CACHE_LIMIT = 16
_fmap_cache: list = []   # [(source object, converted FeatureMap)], most recent last


def set_arithmetic(strict: bool = True) -> None:
    """Reference-exact (strict, default) or fast tensor-core arithmetic."""
    _ARITH["strict"] = bool(strict)


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("corrvol_b200.compat runs on CUDA only; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _backend_ok(backend: Optional[str]) -> None:
    # the reference's names for "pick the best lane" plus this build's lane;
    # anything else is an unknown backend, exactly as _backend.py:69 raises
    _backend.resolve_backend(backend)


def _fmap(x) -> FeatureMap:
    if isinstance(x, FeatureMap):
        return x
    for src, conv in _fmap_cache:
        if src is x:
            return conv
    vals = torch.from_numpy(np.ascontiguousarray(np.asarray(x.values, dtype=np.float32)))
    conv = FeatureMap(vals.to(_device()), check=False)
    _fmap_cache.append((x, conv))
    del _fmap_cache[:-_CACHE_LIMIT]
    return conv


def _cents(c) -> CentroidField:
    if isinstance(c, CentroidField):
        return c
    coords = torch.from_numpy(np.ascontiguousarray(np.asarray(c.coords, dtype=np.float64)))
    return CentroidField(coords.to(_device()), check=False)


def _spec(s) -> LookupSpec:
    if isinstance(s, LookupSpec):
        return s
    return LookupSpec(int(s.radius), int(s.levels), bool(s.normalize))


@dataclass
class HostCostMaps:
    """CostMaps with host numpy values [H, W, L, 2r+1, 2r+1] (types.py:168-200)."""

    values: np.ndarray
    radius: int

    @property
    def height(self) -> int:
        return self.values.shape[0]

    @property
    def width(self) -> int:
        return self.values.shape[1]

    @property
    def levels(self) -> int:
        return self.values.shape[2]

    @property
    def window(self) -> int:
        return 2 * self.radius + 1


def _host(cm) -> HostCostMaps:
    return HostCostMaps(values=cm.values.detach().cpu().numpy(), radius=cm.radius)


# ---- the reference's function names ------------------------------------------

def get_kernels(backend: Optional[str] = None):
    """Kernel lane (_backend.py:59-69); its `.name` is "cuda"."""
    return _backend.get_kernels(backend)


def available_backends() -> list:
    return _backend.available_backends()


def build_feature_pyramid(f2, levels: int) -> FeaturePyramid:
    """dense.py:71-86 (GPU pyramid; level `.values` are CUDA tensors)."""
    return dense.build_feature_pyramid(_fmap(f2), levels)


def build_volume_pyramid(f1, f2, levels: int, mode: str = "pool_volume",
                         backend: Optional[str] = None, counter=None):
    """dense.py:121-160."""
    _backend_ok(backend)
    return dense.build_volume_pyramid(_fmap(f1), _fmap(f2), levels, mode=mode, counter=counter,
                                      strict=_ARITH["strict"])


def lookup_dense(vol, centroids, spec) -> HostCostMaps:
    """dense.py:188-223."""
    return _host(dense.lookup_dense(vol, _cents(centroids), _spec(spec),
                                    strict=_ARITH["strict"]))


def lookup_on_demand(f1, pyr, centroids, spec, backend: Optional[str] = None,
                     counter=None) -> HostCostMaps:
    """ondemand.py:26-90."""
    _backend_ok(backend)
    if not isinstance(pyr, FeaturePyramid):
        pyr = FeaturePyramid([_fmap(l) for l in pyr.levels])
    return _host(ondemand.lookup_on_demand(_fmap(f1), pyr, _cents(centroids), _spec(spec),
                                           counter=counter, strict=_ARITH["strict"]))


def init_state(f1, f2, spec, block: int = 8, cache_cap_bytes: Optional[int] = None,
               hard_limit_bytes: Optional[int] = None, growth_factor: int = 2,
               cache_enabled: bool = True, backend: Optional[str] = None):
    """sparse.py:205-248: the tile-path state with the reference's counters."""
    _backend_ok(backend)
    return sparse.init_state(_fmap(f1), _fmap(f2), _spec(spec), block,
                             cache_cap_bytes=cache_cap_bytes, hard_limit_bytes=hard_limit_bytes,
                             growth_factor=growth_factor, cache_enabled=cache_enabled,
                             mode="tile", strict=_ARITH["strict"], ref_counters=True)


def sample_iteration(state, centroids) -> HostCostMaps:
    """sparse.py:411-452."""
    return _host(sparse.sample_iteration(state, _cents(centroids)))


def memory_footprint(state) -> dict:
    """sparse.py:455-496 (this build's resident bytes, same keys)."""
    return sparse.memory_footprint(state)


#: names a reference module binds to route its calls here
EXPORTS = ("get_kernels", "available_backends", "build_feature_pyramid", "build_volume_pyramid",
           "lookup_dense", "lookup_on_demand", "init_state", "sample_iteration",
           "memory_footprint")
