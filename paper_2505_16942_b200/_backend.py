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

import functools
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


def stream_handle(device=None) -> int:
    """cudaStream_t of the current stream of `device` (default: current device).

    Entry points run under `on_device`, which makes the tensors' device the
    current one, so the library's cudaGetDevice-based choices (shared-memory
    opt-in, SM count) and this stream always match the data.
    """
    return torch.cuda.current_stream(device).cuda_stream


def _device_of(obj):
    """The CUDA device of a tensor / FeatureMap / CentroidField / state, or None."""
    if isinstance(obj, torch.Tensor):
        return obj.device if obj.is_cuda else None
    if isinstance(obj, (list, tuple)):
        return _device_of(obj[0]) if obj else None
    dev = getattr(obj, "device", None)
    if isinstance(dev, torch.device) and dev.type == "cuda":
        return dev
    for attr in ("values", "coords"):
        t = getattr(obj, attr, None)
        if isinstance(t, torch.Tensor) and t.is_cuda:
            return t.device
    lv = getattr(obj, "levels", None)
    if isinstance(lv, (list, tuple)) and lv:
        return _device_of(lv[0])
    return None


class _DeviceGuard:
    """Make `index` the current CUDA device for the duration (no-op when it is)."""

    __slots__ = ("index", "prev")

    def __init__(self, index):
        self.index = index
        self.prev = None

    def __enter__(self):
        if self.index is not None:
            cur = torch.cuda.current_device()
            if cur != self.index:
                self.prev = cur
                torch.cuda.set_device(self.index)
        return self

    def __exit__(self, *exc):
        if self.prev is not None:
            torch.cuda.set_device(self.prev)
        return False


def on_device(fn):
    """Run `fn` with the device of its first CUDA argument current, so kernels
    launch on that device's current stream (a sampler built on cuda:1 never
    launches on cuda:0's stream)."""

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        dev = None
        for a in list(args) + list(kwargs.values()):
            dev = _device_of(a)
            if dev is not None:
                break
        with _DeviceGuard(None if dev is None else dev.index):
            return fn(*args, **kwargs)

    return wrapper


def _flags(strict: bool) -> int:
    return _lib.CVB_STRICT if strict else 0


@on_device
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


@on_device
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


@on_device
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


@on_device
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
