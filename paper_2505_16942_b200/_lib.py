"""ctypes binding of libcorrvol_b200.so (the C-ABI in include/corrvol_b200.h).

This plays the role of the reference's kernel lane selector
(corrvol/_backend.py:1-69): it resolves the compiled lane once and exposes its
functions.  Unlike the reference there is exactly one lane — the sm_100a CUDA
library — and no fallback: if the library is missing or no CUDA device is
present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .types import CacheLimitError, GatherMissError

LIB_PATH = Path(__file__).resolve().parent / "libcorrvol_b200.so"

CVB_OK = 0
CVB_ERR_INVALID = 1
CVB_ERR_GATHER_MISS = 2
CVB_ERR_CACHE_LIMIT = 3
CVB_ERR_CUDA = 4

CVB_STRICT = 1
CVB_COORDS_F64 = 2
CVB_NO_CACHE = 4
CVB_PREP_POOL = 8
CVB_OUT_RAFT = 16
CVB_ACCESS_NO_TRIM = 32
CVB_TC_PAIRS = 64

MAX_LEVELS = 8
TILE_H = 8
TILE_W = 8
META_INTS = 8

_p = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_f32 = C.c_float
_u64p = C.POINTER(C.c_ulonglong)


class PartialDesc(C.Structure):
    """Mirror of cvb_partial_desc."""

    _fields_ = [
        ("h1", _i32), ("w1", _i32), ("d", _i32),
        ("levels", _i32), ("radius", _i32),
        ("th", _i32 * MAX_LEVELS), ("tw", _i32 * MAX_LEVELS),
        ("cap_h", _i32 * MAX_LEVELS), ("cap_w", _i32 * MAX_LEVELS),
        ("tile_begin", _i32), ("tile_end", _i32),
        ("batch", _i32),
    ]


# name -> (restype, argtypes); every symbol declared in include/corrvol_b200.h
SIGNATURES = {
    "cvb_abi_version": (C.c_int, []),
    "cvb_last_error": (C.c_char_p, []),
    "cvb_launch_count": (C.c_ulonglong, []),
    "cvb_corr_pairs": (C.c_int, [_p, _i64, _p, _i64, _i32, _p, _i32, _p]),
    "cvb_corr_gather": (C.c_int, [_p, _i64, _p, _i64, _i32, _p, _p, _p, _i32, _p]),
    "cvb_block_mmm": (C.c_int, [_p, _p, _i64, _i32, _i32, _i32, _p, _i32, _p]),
    "cvb_pool2x2": (C.c_int, [_p, _i32, _i32, _i32, _p, _p]),
    "cvb_build_pyramid": (C.c_int, [_p, _i32, _i32, _i32, _i32, C.POINTER(_p), _p]),
    "cvb_level_floors": (C.c_int, [_p, _i64, _i32, _i32, _p, _p, _p, _p, _p]),
    "cvb_support_valid": (C.c_int, [_p, _i64, _i32, _i32, _i32, _i32, _i32, _p, _p]),
    "cvb_pool_volume": (C.c_int, [_p, _i64, _i32, _i32, _p, _p]),
    "cvb_lookup_dense": (C.c_int, [_p, _i32, _i32, _i32, _i32, _p, _i32, _i32, _i32, _f32,
                                   _p, _i32, _p]),
    "cvb_lookup_on_demand": (C.c_int, [_p, _i32, _i32, _i32, _p, _i32, _i32, _p, _i32, _i32,
                                       _i32, _f32, _p, _p, _i32, _p]),
    "cvb_partial_sizes": (C.c_int, [C.POINTER(PartialDesc), C.POINTER(_i64), C.POINTER(_i64),
                                    C.POINTER(_i64)]),
    "cvb_partial_reset": (C.c_int, [C.POINTER(PartialDesc), _p, _p]),
    "cvb_partial_sample": (C.c_int, [C.POINTER(PartialDesc), _p, C.POINTER(_p), _p, _f32, _p,
                                     C.POINTER(_p), _p, _p, _i32, _p]),
    "cvb_partial_contract": (C.c_int, [C.POINTER(PartialDesc), _p, C.POINTER(_p), _p, _p,
                                       C.POINTER(_p), _p, _i32, _p]),
    "cvb_partial_gather": (C.c_int, [C.POINTER(PartialDesc), _p, C.POINTER(_p), _p, _f32, _p,
                                     C.POINTER(_p), _p, _i32, _p]),
    "cvb_tc_sizes": (C.c_int, [C.POINTER(PartialDesc), C.POINTER(_i64), C.POINTER(_i64)]),
    "cvb_tc_prepare": (C.c_int, [C.POINTER(PartialDesc), _p, C.POINTER(_p), _p, C.POINTER(_p),
                                 _i32, _p]),
    "cvb_partial_contract_tc": (C.c_int, [C.POINTER(PartialDesc), _p, C.POINTER(_p), _p,
                                          C.POINTER(_p), _p, _p, C.POINTER(_p), _p, _i32, _p]),
    "cvb_dense_tc_workspace": (_i64, [C.POINTER(PartialDesc)]),
    "cvb_dense_tc": (C.c_int, [C.POINTER(PartialDesc), _p, C.POINTER(_p), _p, C.POINTER(_p), _p]),
    "cvb_access_union": (C.c_int, [C.POINTER(_p), _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                                   _p, _p]),
    "cvb_access_blocks": (C.c_int, [_p, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _p,
                                    _i64, _p]),
    "cvb_resample_dims": (C.c_int, [_i32, _i32, C.c_double, C.POINTER(_i32), C.POINTER(_i32)]),
    "cvb_resample_flow": (C.c_int, [_p, _i32, _i32, C.c_double, _p, _i32, _i32, _p]),
    "cvb_computation_mask": (C.c_int, [_p, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _p,
                                       _i64, _p]),
    "cvb_mask_accumulate": (C.c_int, [_p, _p, _p, _i64, _i32, _p, _p, _p]),
    "cvb_block_indices_workspace": (_i64, [_i64]),
    "cvb_block_indices": (C.c_int, [_p, _p, _i64, _i64, _i64, _i64, _p, _p, _i64, _p, _p, _p]),
    "cvb_sampled_block_mmm": (C.c_int, [_p, _i32, _i32, _i32, _p, _i32, _i32, _i32, _i32, _i32,
                                        _i64, _p, _i64, _p, _i64, _i32, _p]),
    "cvb_block_gather_sample": (C.c_int, [_p, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                                          _i32, _i32, _i64, _p, _p, _f32, _p, _p, _i32, _p]),
}

_LIB = None


class NativeLibraryError(RuntimeError):
    """The sm_100a library is missing or unusable (there is no CPU fallback)."""


def load(path: os.PathLike | None = None) -> C.CDLL:
    """Load (once) and bind the library; raises NativeLibraryError if absent."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise NativeLibraryError(
            f"{p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.cvb_abi_version() != 2:
        raise NativeLibraryError("ABI version mismatch")
    if path is None:
        _LIB = lib
    return lib


def check(status: int) -> None:
    """Map a cvb_status to the reference's exception types (types.py:27-40)."""
    if status == CVB_OK:
        return
    msg = (load().cvb_last_error() or b"").decode(errors="replace")
    if status == CVB_ERR_INVALID:
        raise ValueError(msg)
    if status == CVB_ERR_GATHER_MISS:
        raise GatherMissError(msg)
    if status == CVB_ERR_CACHE_LIMIT:
        raise CacheLimitError(msg)
    raise RuntimeError(f"CUDA error in libcorrvol_b200: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def ptr(t) -> int:
    """Device pointer of a torch tensor (None -> NULL)."""
    return 0 if t is None else t.data_ptr()


def ptr_array(tensors) -> "C.Array":
    arr = (_p * len(tensors))()
    for i, t in enumerate(tensors):
        arr[i] = ptr(t)
    return arr


def launch_count() -> int:
    return int(load().cvb_launch_count())
