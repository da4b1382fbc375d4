"""Dense variant and the shared pyramid builder (mirrors corrvol/dense.py).

build_feature_pyramid is north-star subsystem (1): one float4 HBM-bound pool
kernel per level, bit-exact with pool2x2 (_pykernels.py:65-81).  The dense
variant materialises [P1, P2_l] per level on the GPU (comparison baseline;
at 8K it reports OOM the way the reference bench does, harness.py:330-333).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

import torch

from . import _lib
from ._backend import on_device, resolve_backend, stream_handle
from .types import (CentroidField, CostMaps, FeatureMap, FeaturePyramid, LookupSpec,
                    WorkCounter, require_cuda)

PYRAMID_MODES = ("pool_volume", "pool_features")


def pooled_dims(shape: Tuple[int, int], level: int) -> Tuple[int, int]:
    """Target grid dims after `level` rounds of 2x2 pooling (dense.py:63-68)."""
    h, w = shape
    for _ in range(level):
        h, w = h // 2, w // 2
    return h, w


def alloc_feature_pyramid(f2: FeatureMap, levels: int) -> FeaturePyramid:
    """Pyramid storage for f2 with levels >= 1 allocated but not yet pooled
    (validation as dense.py:71-86); a fused producer fills them."""
    if levels < 1:
        raise ValueError("levels must be >= 1")
    fh, fw = pooled_dims((f2.height, f2.width), levels - 1)
    if fh < 1 or fw < 1:
        raise ValueError(
            f"pyramid of {levels} levels on {f2.height}x{f2.width} would produce an empty level")
    require_cuda(f2.values)
    maps = [f2]
    for lvl in range(1, levels):
        h, w = pooled_dims((f2.height, f2.width), lvl)
        maps.append(FeatureMap(values=torch.empty((h, w, f2.dims), dtype=torch.float32,
                                                  device=f2.values.device), check=False))
    return FeaturePyramid(levels=maps)


@on_device
def build_feature_pyramid(f2: FeatureMap, levels: int) -> FeaturePyramid:
    """L-level pyramid of f2 (dense.py:71-86)."""
    pyr = alloc_feature_pyramid(f2, levels)
    outs = [m.values for m in pyr.levels]
    _lib.call("cvb_build_pyramid", _lib.ptr(f2.values), f2.height, f2.width, f2.dims, levels,
              _lib.ptr_array(outs), stream_handle())
    return pyr


def _tc_ok(f1: FeatureMap, strict: bool) -> bool:
    return not strict and f1.dims <= 256 and f1.height * f1.width > 0


def _dense_tc(f1: FeatureMap, maps: List[FeatureMap]) -> List[torch.Tensor]:
    """All-pairs matrices [H1*W1, h*w] of f1 against each map, on tcgen05
    (split-fp16, the partial path's accuracy; csrc/partial_tc.cu cvb_dense_tc)."""
    desc = _lib.PartialDesc()
    desc.h1, desc.w1, desc.d = f1.height, f1.width, f1.dims
    desc.levels, desc.radius = len(maps), 0
    for l, m in enumerate(maps):
        if m.dims != f1.dims:
            raise ValueError(f"feature dims differ: {f1.dims} vs {m.dims}")
        desc.th[l], desc.tw[l] = m.height, m.width
        desc.cap_h[l] = desc.cap_w[l] = 1
    dev = f1.values.device
    f1b = _lib.C.c_int64()
    per = (_lib.C.c_int64 * _lib.MAX_LEVELS)()
    _lib.call("cvb_tc_sizes", _lib.C.byref(desc), _lib.C.byref(f1b), per)
    f1s = torch.empty(f1b.value, dtype=torch.uint8, device=dev)
    f2s = [torch.empty(per[l], dtype=torch.uint8, device=dev) for l in range(len(maps))]
    _lib.call("cvb_tc_prepare", _lib.C.byref(desc), _lib.ptr(f1.values),
              _lib.ptr_array([m.values for m in maps]), _lib.ptr(f1s), _lib.ptr_array(f2s), 0,
              stream_handle())
    ws = torch.empty(int(_lib.load().cvb_dense_tc_workspace(_lib.C.byref(desc))),
                     dtype=torch.uint8, device=dev)
    outs = [torch.empty((f1.height * f1.width, m.height * m.width), dtype=torch.float32,
                        device=dev) for m in maps]
    _lib.call("cvb_dense_tc", _lib.C.byref(desc), _lib.ptr(f1s), _lib.ptr_array(f2s),
              _lib.ptr(ws), _lib.ptr_array(outs), stream_handle())
    return outs


@on_device
def build_dense_volume(f1: FeatureMap, f2: FeatureMap, backend: Optional[str] = None,
                       counter: Optional[WorkCounter] = None, strict: bool = False
                       ) -> torch.Tensor:
    """Level-0 all-pairs matrix [H1*W1, H2*W2] float32 (dense.py:27-45).

    strict: the reference's fp32 sequential dots (SIMT, bitwise); otherwise
    tcgen05 split-fp16 (D <= 256) within the fp32 gates."""
    resolve_backend(backend)
    if f1.dims != f2.dims:
        raise ValueError(f"feature dims differ: {f1.dims} vs {f2.dims}")
    require_cuda(f1.values, f2.values)
    if _tc_ok(f1, strict):
        out = _dense_tc(f1, [f2])[0]
        if counter is not None:
            counter.add_dots(out.shape[0] * out.shape[1], f1.dims)
        return out
    a, b = f1.flat(), f2.flat()
    out = torch.empty((a.shape[0], b.shape[0]), dtype=torch.float32, device=a.device)
    _lib.call("cvb_corr_pairs", _lib.ptr(a), a.shape[0], _lib.ptr(b), b.shape[0], f1.dims,
              _lib.ptr(out), _lib.CVB_STRICT if strict else 0, stream_handle())
    if counter is not None:
        counter.add_dots(out.shape[0] * out.shape[1], f1.dims)
    return out


@on_device
def pool_volume(mat: torch.Tensor, tgt_shape: Tuple[int, int]) -> torch.Tensor:
    """2x2 pooling of the volume's target dims (dense.py:48-60)."""
    th, tw = tgt_shape
    if mat.shape[1] != th * tw:
        raise ValueError(f"matrix has {mat.shape[1]} target cells, expected {th}x{tw}")
    if th // 2 == 0 or tw // 2 == 0:
        raise ValueError(f"cannot 2x2-pool dims {(th, tw)}; both must be >= 2")
    require_cuda(mat)
    out = torch.empty((mat.shape[0], (th // 2) * (tw // 2)), dtype=torch.float32,
                      device=mat.device)
    _lib.call("cvb_pool_volume", _lib.ptr(mat), mat.shape[0], th, tw, _lib.ptr(out),
              stream_handle())
    return out


@dataclass
class DenseCorrelationVolume:
    """Precomputed multi-level volume (dense.py:89-108)."""

    src_shape: Tuple[int, int]
    dims: int
    level_mats: List[torch.Tensor]
    level_shapes: List[Tuple[int, int]]
    mode: str

    @property
    def levels(self) -> int:
        return len(self.level_mats)

    def nbytes(self) -> int:
        return sum(m.numel() * 4 for m in self.level_mats)


def estimate_dense_bytes(src_shape: Tuple[int, int], tgt_shape: Tuple[int, int],
                         levels: int) -> int:
    """float32 bytes a dense volume would need (dense.py:111-118)."""
    p1 = src_shape[0] * src_shape[1]
    total = 0
    for lvl in range(levels):
        th, tw = pooled_dims(tgt_shape, lvl)
        total += 4 * p1 * th * tw
    return total


@on_device
def build_volume_pyramid(f1: FeatureMap, f2: FeatureMap, levels: int, mode: str = "pool_volume",
                         backend: Optional[str] = None, counter: Optional[WorkCounter] = None,
                         strict: bool = False) -> DenseCorrelationVolume:
    """Dense volume with an L-level pooled pyramid (dense.py:121-160)."""
    if mode not in PYRAMID_MODES:
        raise ValueError(f"mode must be one of {PYRAMID_MODES}, got {mode!r}")
    fh, fw = pooled_dims((f2.height, f2.width), levels - 1)
    if fh < 1 or fw < 1:
        raise ValueError(
            f"{levels}-level volume on target {f2.height}x{f2.width} would have an empty level")
    mats = [build_dense_volume(f1, f2, backend=backend, counter=counter, strict=strict)]
    shapes = [(f2.height, f2.width)]
    if mode == "pool_volume":
        for _ in range(1, levels):
            mats.append(pool_volume(mats[-1], shapes[-1]))
            shapes.append(pooled_dims(shapes[-1], 1))
    else:
        pyr = build_feature_pyramid(f2, levels)
        if _tc_ok(f1, strict) and levels > 1:  # levels 1.. in one tcgen05 launch
            mats += _dense_tc(f1, pyr.levels[1:])
            for fmap in pyr.levels[1:]:
                shapes.append((fmap.height, fmap.width))
                if counter is not None:
                    counter.add_dots(f1.height * f1.width * fmap.height * fmap.width, f1.dims)
        for lvl in range(len(mats), levels):
            fmap = pyr.levels[lvl]
            mats.append(build_dense_volume(f1, fmap, backend=backend, counter=counter,
                                           strict=strict))
            shapes.append((fmap.height, fmap.width))
    return DenseCorrelationVolume(src_shape=(f1.height, f1.width), dims=f1.dims,
                                  level_mats=mats, level_shapes=shapes, mode=mode)


def coords_flags(centroids: CentroidField, strict: bool) -> int:
    f = _lib.CVB_COORDS_F64 if centroids.is_f64 else 0
    return f | (_lib.CVB_STRICT if strict else 0)


@on_device
def lookup_dense(vol: DenseCorrelationVolume, centroids: CentroidField, spec: LookupSpec,
                 strict: bool = False, out: Optional[torch.Tensor] = None) -> CostMaps:
    """Bilinear (2r+1)^2 windows from the dense volume (dense.py:188-223)."""
    h1, w1 = vol.src_shape
    if (centroids.height, centroids.width) != (h1, w1):
        raise ValueError(
            f"centroid grid {centroids.height}x{centroids.width} does not cover source {h1}x{w1}")
    if spec.levels > vol.levels:
        raise ValueError(f"lookup wants {spec.levels} levels, volume has {vol.levels}")
    require_cuda(centroids.coords, *vol.level_mats)
    k1 = spec.window
    if out is None:
        out = torch.empty((h1, w1, spec.levels, k1, k1), dtype=torch.float32,
                          device=centroids.coords.device)
    scale = spec.scale(vol.dims)
    flags = coords_flags(centroids, strict)
    for lvl in range(spec.levels):
        th, tw = vol.level_shapes[lvl]
        _lib.call("cvb_lookup_dense", _lib.ptr(vol.level_mats[lvl]), h1, w1, th, tw,
                  _lib.ptr(centroids.coords), lvl, spec.levels, spec.radius, scale,
                  _lib.ptr(out), flags, stream_handle())
    return CostMaps(values=out, radius=spec.radius)
