"""Cascaded-init flow resample on the GPU.

Mirrors `resample_flow` / `cascaded_init` (flowio.py:151-199) on CUDA flow
tensors `[H, W, 2]` (x, y); bit-identical to the reference (fp64 arithmetic
with the reference's association, csrc/resample.cu).
"""

from __future__ import annotations

import math

import torch

from . import _lib
from ._backend import on_device, stream_handle
from .types import require_cuda


@on_device
def resample_flow(vectors: torch.Tensor, scale: float) -> torch.Tensor:
    """Bilinearly resample a [H, W, 2] float32 flow field to round(dim*scale)
    (half-up) dims with edge clamping, magnitudes multiplied by scale."""
    if vectors.dim() != 3 or vectors.shape[-1] != 2:
        raise ValueError(f"flow must be [H, W, 2], got {tuple(vectors.shape)}")
    if not (isinstance(scale, (int, float)) and math.isfinite(scale) and scale > 0):
        raise ValueError(f"scale must be a positive finite number, got {scale!r}")
    require_cuda(vectors)
    v = vectors.to(torch.float32).contiguous()
    h, w = v.shape[:2]
    oh, ow = _lib.C.c_int32(), _lib.C.c_int32()
    _lib.call("cvb_resample_dims", h, w, float(scale), _lib.C.byref(oh), _lib.C.byref(ow))
    out = torch.empty((oh.value, ow.value, 2), dtype=torch.float32, device=v.device)
    _lib.call("cvb_resample_flow", _lib.ptr(v), h, w, float(scale), _lib.ptr(out), oh.value,
              ow.value, stream_handle())
    return out


def cascaded_init(low_res_flow: torch.Tensor) -> torch.Tensor:
    """Initial 1/8-grid flow of a full-resolution pass from a 1/4-resolution
    pass's output: one half-scale resample (flowio.py:187-199)."""
    return resample_flow(low_res_flow, 0.5)
