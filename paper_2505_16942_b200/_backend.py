"""Kernel lane: the GPU replacement of corrvol/_backend.py + _ckernels.pyx.

`get_kernels(backend)` returns a namespace with the reference lane's function
names (corr_pairs, corr_gather, block_mmm, pool2x2; _backend.py:26-40).  They
take and return CUDA tensors; like the compiled reference lane they allocate
their outputs.  `strict=True` reproduces the reference arithmetic bit for bit
(fp32 ascending-channel dots without FMA); the default fast lane uses FFMA.
Only one backend exists: None/"auto"/"cuda"; anything else raises ValueError
exactly like the reference's unknown-backend check (_backend.py:69).
"""

from __future__ import annotations

import os
import types
from typing import Optional

import torch

from . import _lib
from .types import require_cuda

BACKENDS = ("cuda",)


def available_backends() -> list:
    return list(BACKENDS)


def default_backend() -> str:
    env = os.environ.get("CORRVOL_BACKEND", "auto").strip().lower()
    if env in ("", "auto", "cuda"):
        return "cuda"
    raise ValueError(f"CORRVOL_BACKEND must be auto or cuda; got {env!r}")


def resolve_backend(backend: Optional[str]) -> str:
    if backend is None or backend == "auto":
        return default_backend()
    if backend != "cuda":
        raise ValueError(f"unknown backend {backend!r}")
    return backend


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def _flags(strict: bool) -> int:
    return _lib.CVB_STRICT if strict else 0


def corr_pairs(a: torch.Tensor, b: torch.Tensor, strict: bool = False) -> torch.Tensor:
    """[n, D] x [m, D] -> [n, m] float32 dots (_ckernels.pyx:17-32)."""
    require_cuda(a, b)
    if a.shape[1] != b.shape[1]:
        raise ValueError(f"channel counts differ: {a.shape[1]} vs {b.shape[1]}")
    a = a.contiguous().float()
    b = b.contiguous().float()
    out = torch.empty((a.shape[0], b.shape[0]), dtype=torch.float32, device=a.device)
    _lib.call("cvb_corr_pairs", _lib.ptr(a), a.shape[0], _lib.ptr(b), b.shape[0], a.shape[1],
              _lib.ptr(out), _flags(strict), stream_handle())
    return out


def corr_gather(f1: torch.Tensor, f2: torch.Tensor, idx: torch.Tensor, valid: torch.Tensor,
                strict: bool = False) -> torch.Tensor:
    """out[p] = valid[p] ? dot(f1[p], f2[idx[p]]) : 0 (_ckernels.pyx:35-52)."""
    require_cuda(f1, f2, idx, valid)
    if f1.shape[1] != f2.shape[1]:
        raise ValueError(f"channel counts differ: {f1.shape[1]} vs {f2.shape[1]}")
    f1 = f1.contiguous().float()
    f2 = f2.contiguous().float()
    idx = idx.contiguous().to(torch.int64)
    valid = valid.contiguous().to(torch.uint8)
    out = torch.empty(f1.shape[0], dtype=torch.float32, device=f1.device)
    _lib.call("cvb_corr_gather", _lib.ptr(f1), f1.shape[0], _lib.ptr(f2), f2.shape[0],
              f1.shape[1], _lib.ptr(idx), _lib.ptr(valid), _lib.ptr(out), _flags(strict),
              stream_handle())
    return out


def block_mmm(at: torch.Tensor, bt: torch.Tensor, strict: bool = False) -> torch.Tensor:
    """[k, n, D] x [k, m, D] -> [k, n, m] (_ckernels.pyx:55-70)."""
    require_cuda(at, bt)
    if at.shape[2] != bt.shape[2] or at.shape[0] != bt.shape[0]:
        raise ValueError("block_mmm operand shapes differ")
    at = at.contiguous().float()
    bt = bt.contiguous().float()
    k, n, d = at.shape
    m = bt.shape[1]
    out = torch.empty((k, n, m), dtype=torch.float32, device=at.device)
    _lib.call("cvb_block_mmm", _lib.ptr(at), _lib.ptr(bt), k, n, m, d, _lib.ptr(out),
              _flags(strict), stream_handle())
    return out


def pool2x2(arr: torch.Tensor) -> torch.Tensor:
    """2x2/stride-2 average pool with floor dims, bit-exact (_pykernels.py:65-81)."""
    require_cuda(arr)
    squeeze = arr.dim() == 2
    a = arr.unsqueeze(-1) if squeeze else arr
    a = a.contiguous().float()
    h, w, d = a.shape
    if h // 2 == 0 or w // 2 == 0:
        raise ValueError(f"cannot 2x2-pool dims {(h, w)}; both must be >= 2")
    out = torch.empty((h // 2, w // 2, d), dtype=torch.float32, device=a.device)
    _lib.call("cvb_pool2x2", _lib.ptr(a), h, w, d, _lib.ptr(out), stream_handle())
    return out.squeeze(-1) if squeeze else out


_LANE = types.SimpleNamespace(name="cuda", corr_pairs=corr_pairs, corr_gather=corr_gather,
                              block_mmm=block_mmm, pool2x2=pool2x2)


def get_kernels(backend: Optional[str] = None) -> types.SimpleNamespace:
    resolve_backend(backend)
    return _LANE
