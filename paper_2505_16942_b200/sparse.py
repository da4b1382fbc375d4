"""Partial (incremental) sampler — the north-star path (mirrors corrvol/sparse.py).

Two interchangeable state layouts behind the reference's API
(init_state / sample_iteration / memory_footprint, sparse.py:205-496):

mode="tile" (default, the B200 design): per 8x8 query tile and level, a
  window-union tiler, a dense contraction of only the newly uncovered cells
  of the tile's support bounding box, a toroidal tile cache in HBM, and a
  shared-memory gather/bilinear sampler — two kernels per iteration
  (csrc/partial.cu), no host synchronisation.

mode="block" (the paper's own pipeline, bit-for-bit the reference state):
  mask scatter -> incremental block ids (prefix sum) -> sampled block MMM
  into a device BlockStore arena with the reference growth/cap/hard-limit
  policy -> proxy gather + combine (csrc/blocks.cu).  Exposes mask_cum,
  mask_union, block_ids, store.used and blocks_computed exactly as the
  reference does; one host sync per level to size the store.

Both return CostMaps bit-identical to the reference with strict=True.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

from . import _lib
from ._backend import on_device, resolve_backend, stream_handle
from .dense import alloc_feature_pyramid, build_feature_pyramid, coords_flags, pooled_dims
from .types import (CacheLimitError, CentroidField, CostMaps, FeatureMap, FeaturePyramid,
                    GatherMissError, LookupSpec, WorkCounter, require_cuda)

#: Default cap on over-allocation beyond current need, per level (5 GiB), sparse.py:45.
DEFAULT_CACHE_CAP_BYTES = 5 * 2 ** 30

_STEPS = ("mask", "indices", "mmm", "cache", "sampling")
MODES = ("tile", "block")

#: Default toroidal cache window (cells per axis) per level for 8x8 query tiles.
#: An 8x8 tile's support box is >= (8/2^l + 2r+1) cells per axis; the window
#: leaves room for flow divergence.  Boxes that do not fit are evaluated
#: directly for that iteration (never wrong, only slower).  34/22 hold the
#: largest box of every BASELINE workload (C1-C4 seed 0 and C5 seeds 0-7;
#: widest: C5 seed 7, 33x33 at level 0, 21x21 at level 1); levels >= 2 get
#: the 2r+2+8 floor (18 at r=4).
DEFAULT_TILE_CAPS = (34, 22, 16, 16, 16, 16, 16, 16)


def _default_cache_cap() -> int:
    env = os.environ.get("CORRVOL_CACHE_CAP_BYTES", "").strip()
    if env:
        cap = int(env)
        if cap < 0:
            raise ValueError("CORRVOL_CACHE_CAP_BYTES must be >= 0")
        return cap
    return DEFAULT_CACHE_CAP_BYTES


def padded_extent(size: int, block: int) -> int:
    """Smallest multiple of block >= size (layout.py:26-28)."""
    return block * ((size + block - 1) // block)


@dataclass
class PaddedGrid:
    """Geometry of a patch-major tiling (layout.py:31-62) without the copy.

    The kernels form the zero-padded B x B tiles on the fly from the
    row-major feature map, so only the geometry is kept.
    """

    block: int
    padded_height: int
    padded_width: int
    orig_height: int
    orig_width: int
    dims: int

    @property
    def tiles_y(self) -> int:
        return self.padded_height // self.block

    @property
    def tiles_x(self) -> int:
        return self.padded_width // self.block

    @property
    def n_tiles(self) -> int:
        return self.tiles_y * self.tiles_x

    @classmethod
    def of(cls, h: int, w: int, d: int, block: int) -> "PaddedGrid":
        return cls(block, padded_extent(h, block), padded_extent(w, block), h, w, d)


class BlockStore:
    """Device arena of B^2 x B^2 float32 blocks (sparse.py:61-130).

    Same growth (x growth_factor, capped at need + overalloc_cap) and
    hard-limit policy as the reference; the check happens before any state
    is touched, so a CacheLimitError leaves the sampler state intact
    (the reference mutates mask_cum/block_ids first, sparse.py:436-440).
    """

    def __init__(self, block: int, growth_factor: int = 2,
                 overalloc_cap_bytes: Optional[int] = None,
                 hard_limit_bytes: Optional[int] = None, device=None):
        if growth_factor < 2:
            raise ValueError("growth_factor must be >= 2")
        self.block = block
        self.block_cells = block * block
        self.bytes_per_block = 4 * self.block_cells * self.block_cells
        self.growth_factor = growth_factor
        self.overalloc_cap_bytes = (_default_cache_cap() if overalloc_cap_bytes is None
                                    else overalloc_cap_bytes)
        self.hard_limit_bytes = hard_limit_bytes
        self.device = device if device is not None else torch.device("cpu")
        self.data = torch.empty((0, self.block_cells, self.block_cells), dtype=torch.float32,
                                device=self.device)
        self.used = 0
        self.growth_events = 0

    @property
    def capacity(self) -> int:
        return self.data.shape[0]

    def used_bytes(self) -> int:
        return self.used * self.bytes_per_block

    def capacity_bytes(self) -> int:
        return self.capacity * self.bytes_per_block

    def check_limit(self, k_new: int) -> None:
        needed = self.used + k_new
        if self.hard_limit_bytes is not None and \
                needed * self.bytes_per_block > self.hard_limit_bytes:
            raise CacheLimitError(
                f"block cache needs {needed * self.bytes_per_block} bytes, "
                f"hard limit is {self.hard_limit_bytes}")

    def ensure_capacity(self, k_new: int) -> None:
        self.check_limit(k_new)
        needed = self.used + k_new
        if needed <= self.capacity:
            return
        cap = max(self.capacity, 1)
        while cap < needed:
            cap *= self.growth_factor
        cap_blocks = self.overalloc_cap_bytes // self.bytes_per_block
        cap = min(cap, needed + cap_blocks)
        grown = torch.empty((cap, self.block_cells, self.block_cells), dtype=torch.float32,
                            device=self.device)
        if self.used:
            grown[: self.used].copy_(self.data[: self.used])
        self.data = grown
        self.growth_events += 1

    def append(self, blocks: torch.Tensor) -> int:
        k = blocks.shape[0]
        start = self.used
        self.data[start: start + k] = blocks.to(self.device)
        self.used += k
        return start

    def reset(self) -> None:
        self.used = 0


class _StoreCount:
    """Tile mode with ref_counters: the `store.used` the reference's BlockStore
    would report (blocks of the level held after this iteration), kept on the
    device and synced when read."""

    def __init__(self, counts: torch.Tensor, index: int, bytes_per_block: int):
        self._counts = counts
        self._index = index
        self.bytes_per_block = bytes_per_block

    @property
    def used(self) -> int:
        return int(self._counts[self._index].item())

    def used_bytes(self) -> int:
        return self.used * self.bytes_per_block


class TileWorkCounter(WorkCounter):
    """WorkCounter of a tile-mode state without ref_counters: dot_products /
    macs are the tile path's executed dots; the reference's block currency is
    not tracked, and reading it fails loudly instead of returning 0."""

    def __getattribute__(self, name):
        if name == "blocks_computed":
            raise RuntimeError(
                "blocks_computed is the reference's block-granular work currency; the tile "
                "path tracks it only with init_state(..., ref_counters=True)")
        return super().__getattribute__(name)


_POPC = None


def _popcount_sum(words: torch.Tensor) -> int:
    global _POPC
    if _POPC is None or _POPC.device != words.device:
        _POPC = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int64,
                             device=words.device)
    return int(_POPC[words.contiguous().view(torch.uint8).long()].sum().item())


def unpack_bits(words: torch.Tensor, n: int) -> torch.Tensor:
    """[rows, wpr] uint32-as-int32 bitmask -> [rows, n] bool."""
    shifts = torch.arange(32, device=words.device, dtype=torch.int32)
    bits = (words[:, :, None] >> shifts) & 1
    return bits.reshape(words.shape[0], -1)[:, :n].bool()


@dataclass
class _LevelState:
    """Per-level state (sparse.py:133-150)."""

    tgt_shape: Tuple[int, int]
    pm2: PaddedGrid
    # block mode (reference state), bit-packed masks [n_src, words_per_row]
    mask_cum_bits: Optional[torch.Tensor] = None
    mask_union_bits: Optional[torch.Tensor] = None
    block_ids: Optional[torch.Tensor] = None
    store: Optional[BlockStore] = None
    # tile mode
    cache: Optional[torch.Tensor] = None
    cap: Tuple[int, int] = (0, 0)

    @property
    def n_tgt_tiles(self) -> int:
        return self.pm2.n_tiles

    @property
    def words_per_row(self) -> int:
        return (self.pm2.n_tiles + 31) // 32

    @property
    def mask_cum(self) -> torch.Tensor:
        return unpack_bits(self.mask_cum_bits, self.n_tgt_tiles)

    @property
    def mask_union(self) -> torch.Tensor:
        return unpack_bits(self.mask_union_bits, self.n_tgt_tiles)

    @property
    def block_positions(self) -> int:
        n_src = self.mask_cum_bits.shape[0] if self.mask_cum_bits is not None else 0
        return n_src * self.n_tgt_tiles


class SparseVolumeState:
    """Device state of the partial sampler (sparse.py:153-202).

    Single writer: sample_iteration calls on one state must be serialised
    (stream order), as in the reference (sparse.py:170-173).
    """

    def __init__(self, f1: FeatureMap, spec: LookupSpec, block: int, pm1: PaddedGrid,
                 pyramid: FeaturePyramid, levels: List[_LevelState], cache_enabled: bool,
                 backend: Optional[str], mode: str, strict: bool):
        self.f1 = f1
        self.spec = spec
        self.block = block
        self.pm1 = pm1
        self.pyramid = pyramid
        self.levels = levels
        self.cache_enabled = cache_enabled
        self.backend = backend
        self.mode = mode
        self.strict = strict
        self.iteration = 0
        self.timings: Dict[str, float] = {step: 0.0 for step in _STEPS}
        self._counter = WorkCounter()
        dev = f1.values.device
        self.device = dev
        self._dev_counters = torch.zeros(4, dtype=torch.int64, device=dev)
        self.desc: Optional[_lib.PartialDesc] = None
        self.meta: Optional[torch.Tensor] = None
        self._src_tile = None
        self.tc = False
        self.pipeline_splits = 1
        self._side_stream = None
        self._desc_cache = {}
        self.n_tiles = 0
        self.tc_f1 = None
        self.tc_f2 = None
        self.ref_counters = False
        self._ref_counts = None
        self.batch = 1
        self.scratch_tiles = 0

    # -- reference-compatible attributes ------------------------------------
    @property
    def n_src_tiles(self) -> int:
        return self.pm1.n_tiles

    @property
    def src_tile(self) -> torch.Tensor:
        if self._src_tile is None:
            h, w, b = self.f1.height, self.f1.width, self.block
            p = torch.arange(h * w, device=self.device, dtype=torch.int64)
            ys, xs = p // w, p % w
            self._src_tile = (ys // b) * self.pm1.tiles_x + (xs // b)
        return self._src_tile

    @property
    def src_inner(self) -> torch.Tensor:
        h, w, b = self.f1.height, self.f1.width, self.block
        p = torch.arange(h * w, device=self.device, dtype=torch.int64)
        return ((p // w) % b) * b + (p % w) % b

    @property
    def counter(self) -> WorkCounter:
        """WorkCounter synced from the device (one sync per read).

        Tile mode with ref_counters: the reference's block-model counts
        (blocks_computed; dot_products = blocks * B^4, sparse.py:342-346).
        Tile mode without: the tile path's executed dots, and blocks_computed
        raises (TileWorkCounter)."""
        if self.mode == "tile":
            if self.ref_counters:
                blocks = int(self._ref_counts[0].item())
                b4 = self.block ** 4
                self._counter.blocks_computed = blocks
                self._counter.dot_products = blocks * b4
                self._counter.macs = blocks * b4 * self.f1.dims
                return self._counter
            dots = int(self._dev_counters[0].item())
            c = TileWorkCounter()
            c.dot_products = dots
            c.macs = dots * self.f1.dims
            return c
        return self._counter

    @property
    def device_counters(self) -> Dict[str, int]:
        c = self._dev_counters.tolist()
        return {"dots": c[0], "cells": c[1], "overflow_tile_levels": c[2],
                "empty_tile_levels": c[3]}


def _tile_caps(spec: LookupSpec, tile_caps) -> List[Tuple[int, int]]:
    caps = []
    for lvl in range(spec.levels):
        if tile_caps is None:
            c = DEFAULT_TILE_CAPS[lvl]
            # the cap must at least hold one tile's worth of supports
            c = max(c, 2 * spec.radius + 2 + 8)
            caps.append((c, c))
        else:
            c = tile_caps[lvl] if isinstance(tile_caps, (list, tuple)) else tile_caps
            caps.append((c, c) if isinstance(c, int) else tuple(c))
    return caps


@on_device
def init_state(f1: FeatureMap, f2: FeatureMap, spec: LookupSpec, block: int = 8,
               cache_cap_bytes: Optional[int] = None, hard_limit_bytes: Optional[int] = None,
               growth_factor: int = 2, cache_enabled: bool = True,
               backend: Optional[str] = None, mode: str = "tile", strict: bool = False,
               tile_caps=None, pyramid: Optional[FeaturePyramid] = None,
               tensor_cores: Optional[bool] = None,
               pipeline_splits: Optional[int] = None,
               ref_counters: bool = False,
               scratch_tiles: Optional[int] = None) -> SparseVolumeState:
    """One-time preprocessing for an image pair (sparse.py:205-248).

    Builds the fmap2 pyramid on the GPU and allocates the level states.
    mode="tile": cache window per level from tile_caps (default
    DEFAULT_TILE_CAPS); hard_limit_bytes bounds the preallocated tile cache.
    mode="block": reference block store per level (growth, cap, hard limit).
    tensor_cores (tile mode, fast arithmetic): contract on tcgen05 with
    split-fp16 operands (default when not strict and D <= 256).
    ref_counters (tile mode): also keep the reference's block-granular state
    per iteration on the device — bit-packed mask_cum / mask_union and the
    block counts (counter.blocks_computed, levels[l].store.used,
    mask_union, block_positions) that the reference harness reads
    (harness.py:244-245,406-436) — at one mask kernel + one accumulate kernel
    per level and iteration; off by default so the timed path is not taxed.
    scratch_tiles (tile mode, cache off): keep cache windows for only this many
    tiles and run each iteration as contract+gather over consecutive ranges
    of that many tiles — the stateless recompute ("on-demand") configuration
    with bounded memory.
    """
    resolve_backend(backend)
    if f1.dims != f2.dims:
        raise ValueError(f"feature dims differ: {f1.dims} vs {f2.dims}")
    if block < 1:
        raise ValueError("block must be >= 1")
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    require_cuda(f1.values, f2.values)
    if tensor_cores is None:
        tensor_cores = mode == "tile" and (not strict) and f1.dims <= 256
    if tensor_cores and strict:
        raise ValueError("strict arithmetic runs on the FP32 pipe; tensor_cores=False")
    # on the tensor-core path the operand split builds the pyramid in the same pass
    fuse_pyramid = tensor_cores and mode == "tile" and pyramid is None
    if pyramid is not None:
        pyr = pyramid
    elif fuse_pyramid:
        pyr = alloc_feature_pyramid(f2, spec.levels)
    else:
        pyr = build_feature_pyramid(f2, spec.levels)
    if len(pyr) < spec.levels:
        raise ValueError("pyramid has fewer levels than the spec")
    pm1 = PaddedGrid.of(f1.height, f1.width, f1.dims, block)
    dev = f1.values.device
    levels = []
    for lvl in range(spec.levels):
        fmap = pyr.levels[lvl]
        levels.append(_LevelState(tgt_shape=(fmap.height, fmap.width),
                                  pm2=PaddedGrid.of(fmap.height, fmap.width, fmap.dims, block)))
    state = SparseVolumeState(f1, spec, block, pm1, pyr, levels, cache_enabled, backend, mode,
                              strict)
    if mode == "tile":
        if scratch_tiles is not None and cache_enabled:
            raise ValueError("scratch_tiles needs cache_enabled=False")
        _setup_tile(state, tile_caps, hard_limit_bytes, tensor_cores, fuse_pyramid,
                    pipeline_splits, ref_counters, scratch_tiles=scratch_tiles)
    else:
        for lv in levels:
            n_src, wpr = pm1.n_tiles, lv.words_per_row
            lv.mask_cum_bits = torch.zeros((n_src, wpr), dtype=torch.int32, device=dev)
            lv.mask_union_bits = torch.zeros((n_src, wpr), dtype=torch.int32, device=dev)
            lv.block_ids = torch.full((n_src, lv.n_tgt_tiles), -1, dtype=torch.int64, device=dev)
            lv.store = BlockStore(block, growth_factor=growth_factor,
                                  overalloc_cap_bytes=cache_cap_bytes,
                                  hard_limit_bytes=hard_limit_bytes, device=dev)
    return state


def _setup_tile(state: SparseVolumeState, tile_caps, hard_limit_bytes: Optional[int],
                tensor_cores: bool, fuse_pyramid: bool, pipeline_splits: Optional[int],
                ref_counters: bool, batch: int = 1, pair_height: Optional[int] = None,
                scratch_tiles: Optional[int] = None) -> None:
    """Tile-mode device state: descriptor, metadata, tile caches (all pairs of
    a batch), optional reference-model counters, split operands."""
    spec, levels, dev = state.spec, state.levels, state.device
    if spec.radius > 8:
        raise ValueError("tile mode supports radius <= 8")
    desc = _lib.PartialDesc()
    desc.h1 = state.f1.height if pair_height is None else pair_height
    desc.w1, desc.d = state.f1.width, state.f1.dims
    desc.levels, desc.radius = spec.levels, spec.radius
    desc.batch = batch
    caps = _tile_caps(spec, tile_caps)
    for lvl, lv in enumerate(levels):
        desc.th[lvl], desc.tw[lvl] = lv.tgt_shape
        desc.cap_h[lvl], desc.cap_w[lvl] = caps[lvl]
        lv.cap = caps[lvl]
    n_tiles = _lib.C.c_int64()
    meta_ints = _lib.C.c_int64()
    per_level = (_lib.C.c_int64 * _lib.MAX_LEVELS)()
    _lib.call("cvb_partial_sizes", _lib.C.byref(desc), _lib.C.byref(n_tiles),
              _lib.C.byref(meta_ints), per_level)
    total = 4 * sum(per_level[i] for i in range(spec.levels))
    if hard_limit_bytes is not None and total > hard_limit_bytes:
        raise CacheLimitError(
            f"tile cache needs {total} bytes, hard limit is {hard_limit_bytes}")
    state.desc = desc
    state.batch = batch
    state.n_tiles = n_tiles.value
    state.meta = torch.empty(meta_ints.value, dtype=torch.int32, device=dev)
    if scratch_tiles is not None:
        state.scratch_tiles = max(1, min(int(scratch_tiles), state.n_tiles))
    for lvl, lv in enumerate(levels):
        n = per_level[lvl]
        if state.scratch_tiles:
            n = n // state.n_tiles * state.scratch_tiles
        lv.cache = torch.empty(n, dtype=torch.float32, device=dev)
    _lib.call("cvb_partial_reset", _lib.C.byref(desc), _lib.ptr(state.meta), stream_handle())
    if ref_counters:
        if batch > 1:
            raise ValueError("ref_counters needs a single-pair state")
        state.ref_counters = True
        state._ref_counts = torch.zeros(1 + spec.levels, dtype=torch.int64, device=dev)
        for lvl, lv in enumerate(levels):
            n_src, wpr = state.pm1.n_tiles, lv.words_per_row
            lv.mask_cum_bits = torch.zeros((n_src, wpr), dtype=torch.int32, device=dev)
            lv.mask_union_bits = torch.zeros((n_src, wpr), dtype=torch.int32, device=dev)
            lv.store = _StoreCount(state._ref_counts, 1 + lvl, 4 * state.block ** 4)
    if tensor_cores:
        _prepare_tc(state, pool=fuse_pyramid)
        # overlap contraction and gathering across tile ranges: measured on
        # B200 at C4, no gain (the contraction's shared memory keeps the
        # sampler from co-residing), so off by default
        state.pipeline_splits = max(1, int(pipeline_splits or 1))


@on_device
def init_state_batch(f1: torch.Tensor, f2: torch.Tensor, spec: LookupSpec, strict: bool = False,
                     cache_enabled: bool = True, tile_caps=None,
                     hard_limit_bytes: Optional[int] = None,
                     tensor_cores: Optional[bool] = None) -> SparseVolumeState:
    """One tile-mode state for B image pairs of equal geometry (C5).

    f1, f2: [B, H, W, D] CUDA tensors.  Every iteration is ONE plan, ONE
    contraction and ONE sampler launch over all pairs' tiles (the pair index
    is folded into the tile id, csrc/partial.cuh `tile_ref`); per-pair
    pyramids, caches, metadata and split operands live in pair-major arenas.
    `sample_iteration(state, coords)` takes coords [B*H, W, 2] (a
    [B, H, W, 2] tensor viewed as one tall field) and returns [B*H, W, L,
    2r+1, 2r+1]; `BatchCorrSampler` does the reshaping.  Per pair the
    results are bit-identical to a single-pair state (same kernels, same
    per-query arithmetic)."""
    if f1.dim() != 4 or f1.shape != f2.shape:
        raise ValueError("f1 and f2 must both be [B, H, W, D] with equal shapes")
    require_cuda(f1, f2)
    b, h, w, d = f1.shape
    if tensor_cores is None:
        tensor_cores = (not strict) and d <= 256
    if tensor_cores and strict:
        raise ValueError("strict arithmetic runs on the FP32 pipe; tensor_cores=False")
    f1 = f1.to(torch.float32).contiguous()
    f2 = f2.to(torch.float32).contiguous()
    dev = f1.device
    fh, fw = pooled_dims((h, w), spec.levels - 1)
    if fh < 1 or fw < 1:
        raise ValueError(f"pyramid of {spec.levels} levels on {h}x{w} would produce an empty "
                         "level")
    dims = [pooled_dims((h, w), l) for l in range(spec.levels)]
    lv_t = [f2] + [torch.empty((b, th, tw, d), dtype=torch.float32, device=dev)
                   for th, tw in dims[1:]]
    if not tensor_cores:  # the fused split pools on the tensor-core path
        for i in range(b):
            _lib.call("cvb_build_pyramid", _lib.ptr(f2[i]), h, w, d, spec.levels,
                      _lib.ptr_array([t[i] for t in lv_t]), stream_handle())
    pyr = FeaturePyramid([FeatureMap(t.view(b * t.shape[1], t.shape[2], d), check=False)
                          for t in lv_t])
    pm1 = PaddedGrid.of(h, w, d, 8)
    levels = [_LevelState(tgt_shape=dims[l], pm2=PaddedGrid.of(dims[l][0], dims[l][1], d, 8))
              for l in range(spec.levels)]
    state = SparseVolumeState(FeatureMap(f1.view(b * h, w, d), check=False), spec, 8, pm1, pyr,
                              levels, cache_enabled, None, "tile", strict)
    _setup_tile(state, tile_caps, hard_limit_bytes, tensor_cores, tensor_cores, None, False,
                batch=b, pair_height=h)
    return state


def _prepare_tc(state: SparseVolumeState, pool: bool = False) -> None:
    """Split F1 / the fmap2 pyramid into per-row-scaled fp16 hi/lo operands
    (once per pair); with `pool`, pyramid levels >= 1 are produced in the
    same pass (bit-exact pool2x2)."""
    spec = state.spec
    f1b = _lib.C.c_int64()
    per = (_lib.C.c_int64 * _lib.MAX_LEVELS)()
    _lib.call("cvb_tc_sizes", _lib.C.byref(state.desc), _lib.C.byref(f1b), per)
    dev = state.device
    state.tc_f1 = torch.empty(f1b.value, dtype=torch.uint8, device=dev)
    state.tc_f2 = [torch.empty(per[l], dtype=torch.uint8, device=dev)
                   for l in range(spec.levels)]
    f2s = [state.pyramid.levels[l].values for l in range(spec.levels)]
    _lib.call("cvb_tc_prepare", _lib.C.byref(state.desc), _lib.ptr(state.f1.values),
              _lib.ptr_array(f2s), _lib.ptr(state.tc_f1), _lib.ptr_array(state.tc_f2),
              _lib.CVB_PREP_POOL if pool else 0, stream_handle())
    state.tc = True


def _contract_args(state: SparseVolumeState, centroids: CentroidField, flags: int):
    spec = state.spec
    f2s = _lib.ptr_array([state.pyramid.levels[l].values for l in range(spec.levels)])
    caches = _lib.ptr_array([lv.cache for lv in state.levels])
    return f2s, caches


#: cold iterations (the first, or every one with the cache off) contract on
#: SM pairs (CVB_TC_PAIRS); CVB_TC_PAIRS=0 in the environment turns it off
_PAIRS = os.environ.get("CVB_TC_PAIRS", "1").strip() != "0"


def _contract(state: SparseVolumeState, centroids: CentroidField, flags: int, f2s,
              caches) -> None:
    if state.tc:
        if _PAIRS and (state.iteration == 0 or not state.cache_enabled):
            flags |= _lib.CVB_TC_PAIRS
        _lib.call("cvb_partial_contract_tc", _lib.C.byref(state.desc), _lib.ptr(state.f1.values),
                  f2s, _lib.ptr(state.tc_f1), _lib.ptr_array(state.tc_f2),
                  _lib.ptr(centroids.coords), _lib.ptr(state.meta),
                  caches, _lib.ptr(state._dev_counters), flags, stream_handle())
    else:
        _lib.call("cvb_partial_contract", _lib.C.byref(state.desc), _lib.ptr(state.f1.values),
                  f2s, _lib.ptr(centroids.coords), _lib.ptr(state.meta), caches,
                  _lib.ptr(state._dev_counters), flags, stream_handle())


def _gather(state: SparseVolumeState, centroids: CentroidField, flags: int, f2s, caches,
            out: torch.Tensor) -> None:
    _lib.call("cvb_partial_gather", _lib.C.byref(state.desc), _lib.ptr(state.f1.values), f2s,
              _lib.ptr(centroids.coords), state.spec.scale(state.f1.dims), _lib.ptr(state.meta),
              caches, _lib.ptr(out), flags, stream_handle())


def _level_centroid_floors(state: SparseVolumeState, centroids: CentroidField, level: int):
    """(x0, y0, fx, fy) per query (sparse.py:251-259), computed on the GPU."""
    p = centroids.height * centroids.width
    dev = centroids.coords.device
    x0 = torch.empty(p, dtype=torch.int64, device=dev)
    y0 = torch.empty(p, dtype=torch.int64, device=dev)
    fx = torch.empty(p, dtype=torch.float64, device=dev)
    fy = torch.empty(p, dtype=torch.float64, device=dev)
    _lib.call("cvb_level_floors", _lib.ptr(centroids.coords), p, level,
              coords_flags(centroids, False), _lib.ptr(x0), _lib.ptr(y0), _lib.ptr(fx),
              _lib.ptr(fy), stream_handle())
    return x0, y0, fx, fy


def _check_grid(state: SparseVolumeState, centroids: CentroidField) -> None:
    if (centroids.height, centroids.width) != (state.f1.height, state.f1.width):
        raise ValueError("centroid grid does not cover the source grid")
    require_cuda(centroids.coords)


def _mask_bits(state: SparseVolumeState, centroids: CentroidField, level: int) -> torch.Tensor:
    lv = state.levels[level]
    mask = torch.zeros((state.n_src_tiles, lv.words_per_row), dtype=torch.int32,
                       device=state.device)
    _lib.call("cvb_computation_mask", _lib.ptr(centroids.coords), state.f1.height,
              state.f1.width, level, state.spec.radius, state.block, lv.pm2.padded_height,
              lv.pm2.padded_width, coords_flags(centroids, False), _lib.ptr(mask),
              lv.words_per_row, stream_handle())
    return mask


@on_device
def set_computation_mask(state: SparseVolumeState, centroids: CentroidField,
                         level: int) -> torch.Tensor:
    """This iteration's [n_src_tiles, n_tgt_tiles] bool mask (sparse.py:262-290); pure."""
    _check_grid(state, centroids)
    lv = state.levels[level]
    return unpack_bits(_mask_bits(state, centroids, level), lv.n_tgt_tiles)


def _pack_bits(mask: torch.Tensor, wpr: int) -> torch.Tensor:
    rows, n = mask.shape
    padded = torch.zeros((rows, wpr * 32), dtype=torch.int64, device=mask.device)
    padded[:, :n] = mask.to(torch.int64)
    weights = (torch.ones(32, dtype=torch.int64, device=mask.device)
               << torch.arange(32, device=mask.device, dtype=torch.int64))
    words = (padded.view(rows, wpr, 32) * weights).sum(dim=2)
    return ((words + 2 ** 31) % 2 ** 32 - 2 ** 31).to(torch.int32)


def _block_indices_bits(state: SparseVolumeState, mask_bits: torch.Tensor, level: int):
    """Positions/ids of the newly needed blocks; updates cum/union/ids (sparse.py:293-309)."""
    lv = state.levels[level]
    k = _popcount_sum(mask_bits & ~lv.mask_cum_bits)
    lv.store.check_limit(k)  # transactional: raise before touching state
    n = mask_bits.numel()
    ws = torch.empty(int(_lib.load().cvb_block_indices_workspace(n)), dtype=torch.uint8,
                     device=state.device)
    positions = torch.empty(max(k, 1), dtype=torch.int64, device=state.device)
    count = torch.zeros(1, dtype=torch.int64, device=state.device)
    used = lv.store.used
    _lib.call("cvb_block_indices", _lib.ptr(mask_bits), _lib.ptr(lv.mask_cum_bits),
              mask_bits.shape[0], lv.words_per_row, lv.n_tgt_tiles, used,
              _lib.ptr(lv.block_ids), _lib.ptr(positions), k, _lib.ptr(count), _lib.ptr(ws),
              stream_handle())
    lv.mask_union_bits |= mask_bits
    ids = used + torch.arange(k, dtype=torch.int64, device=state.device)
    return positions[:k], ids


@on_device
def compute_block_indices(state: SparseVolumeState, new_mask: torch.Tensor, level: int):
    """Assign ids to this iteration's newly needed blocks (sparse.py:293-309)."""
    lv = state.levels[level]
    return _block_indices_bits(state, _pack_bits(new_mask.to(state.device), lv.words_per_row),
                               level)


@on_device
def sampled_block_mmm(state: SparseVolumeState, level: int, positions: torch.Tensor,
                      timings=None) -> torch.Tensor:
    """Compute and append the blocks at `positions` (sparse.py:312-346)."""
    lv = state.levels[level]
    k = int(positions.numel())
    b2 = state.block * state.block
    if k == 0:
        return torch.empty((0, b2, b2), dtype=torch.float32, device=state.device)
    lv.store.ensure_capacity(k)
    first = lv.store.used
    fmap = state.pyramid.levels[level]
    _lib.call("cvb_sampled_block_mmm", _lib.ptr(state.f1.values), state.f1.height,
              state.f1.width, state.f1.dims, _lib.ptr(fmap.values), fmap.height, fmap.width,
              state.block, state.pm1.tiles_x, lv.pm2.tiles_x, lv.n_tgt_tiles,
              _lib.ptr(positions.contiguous()), k, _lib.ptr(lv.store.data), first,
              _lib.CVB_STRICT if state.strict else 0, stream_handle())
    lv.store.used += k
    state._counter.blocks_computed += k
    state._counter.add_dots(k * b2 * b2, state.f1.dims)
    return lv.store.data[first: first + k]


@dataclass
class ProxyBlock:
    """(2r+2)^2 patch of exact correlation cells for one source pixel (sparse.py:153-164)."""

    level: int
    anchor_x: int
    anchor_y: int
    values: np.ndarray


def gather_proxy(state: SparseVolumeState, level: int, pixel: int,
                 centroid: Tuple[float, float]) -> ProxyBlock:
    """Proxy patch for one source pixel, block mode (sparse.py:378-408)."""
    if state.mode != "block":
        raise ValueError("gather_proxy needs a block-mode state")
    lv = state.levels[level]
    b, r, k = state.block, state.spec.radius, state.spec.support
    pth, ptw = lv.pm2.padded_height, lv.pm2.padded_width
    x0 = math.floor(centroid[0] / (2 ** level))
    y0 = math.floor(centroid[1] / (2 ** level))
    out = np.zeros((k, k), dtype=np.float32)
    src_tile = int(state.src_tile[pixel].item())
    src_inner = int(state.src_inner[pixel].item())
    ids = lv.block_ids[src_tile].cpu()
    for j in range(k):
        for i in range(k):
            ty, tx = y0 - r + j, x0 - r + i
            if not (0 <= ty < pth and 0 <= tx < ptw):
                continue
            bid = int(ids[(ty // b) * lv.pm2.tiles_x + tx // b])
            if bid < 0:
                raise GatherMissError(
                    f"level {level}: pixel {pixel} needs target cell ({ty}, {tx}) "
                    "whose block was never computed")
            out[j, i] = float(lv.store.data[bid, src_inner, (ty % b) * b + tx % b].item())
    return ProxyBlock(level=level, anchor_x=x0 - r, anchor_y=y0 - r, values=out)


def _sample_block_mode(state: SparseVolumeState, centroids: CentroidField,
                       out: torch.Tensor) -> None:
    spec = state.spec
    scale = spec.scale(state.f1.dims)
    flags = coords_flags(centroids, state.strict)
    if not state.cache_enabled:
        for lv in state.levels:
            lv.mask_cum_bits.zero_()
            lv.block_ids.fill_(-1)
            lv.store.reset()
    # size every level first so a CacheLimitError leaves the state untouched
    masks = [_mask_bits(state, centroids, lvl) for lvl in range(spec.levels)]
    for lvl, lv in enumerate(state.levels):
        lv.store.check_limit(_popcount_sum(masks[lvl] & ~lv.mask_cum_bits))
    miss = torch.zeros(1, dtype=torch.int32, device=state.device)
    for lvl, lv in enumerate(state.levels):
        positions, _ = _block_indices_bits(state, masks[lvl], lvl)
        sampled_block_mmm(state, lvl, positions)
        _lib.call("cvb_block_gather_sample", _lib.ptr(centroids.coords), state.f1.height,
                  state.f1.width, lvl, spec.levels, spec.radius, state.block,
                  lv.pm2.padded_height, lv.pm2.padded_width, state.pm1.tiles_x, lv.pm2.tiles_x,
                  lv.n_tgt_tiles, _lib.ptr(lv.block_ids),
                  _lib.ptr(lv.store.data) if lv.store.capacity else 0, scale, _lib.ptr(out),
                  _lib.ptr(miss), flags, stream_handle())
    if int(miss.item()):
        raise GatherMissError("a proxy gather hit a block that was never computed")


def _accumulate_ref_counters(state: SparseVolumeState, centroids: CentroidField) -> None:
    """The reference's mask / block accounting for one tile-mode iteration
    (set_computation_mask + the counting half of compute_block_indices,
    sparse.py:262-309, with the cache-off reset of :426-430), on the device."""
    counts = state._ref_counts
    for lvl, lv in enumerate(state.levels):
        mask = _mask_bits(state, centroids, lvl)
        _lib.call("cvb_mask_accumulate", _lib.ptr(mask), _lib.ptr(lv.mask_cum_bits),
                  _lib.ptr(lv.mask_union_bits), mask.numel(), 0 if state.cache_enabled else 1,
                  _lib.ptr(counts), counts.data_ptr() + 8 * (1 + lvl), stream_handle())


def _range_descs(state: SparseVolumeState, splits: int):
    """PartialDesc copies covering `splits` contiguous tile ranges."""
    key = ("ranges", splits)
    if state._desc_cache.get(key) is None:
        n = state.n_tiles
        # whole tile rows per range (the cold SM-pair contraction pairs tiles
        # within a row)
        tx = -(-state.f1.width // _lib.TILE_W)
        rows = n // tx
        bounds = sorted(set([tx * (rows * i // splits) for i in range(splits)] + [n]))
        descs = []
        for i in range(len(bounds) - 1):
            d = _lib.PartialDesc()
            _lib.C.pointer(d)[0] = state.desc
            d.tile_begin, d.tile_end = bounds[i], bounds[i + 1]
            descs.append(d)
        state._desc_cache[key] = descs
    return state._desc_cache[key]


def _sample_scratch_ranges(state: SparseVolumeState, centroids: CentroidField, flags: int,
                           out: torch.Tensor) -> None:
    """Cache-off iteration over ranges of `scratch_tiles` tiles: each range is
    contracted into the scratch windows and gathered before the next range
    reuses them (stream order).  The kernels address the cache by global tile
    index, so each range passes the scratch base shifted back by its first
    tile (only offsets inside the scratch are dereferenced)."""
    per_tile = [lv.cache.numel() // state.scratch_tiles for lv in state.levels]
    # ranges of whole tile rows (the cold SM-pair contraction pairs tiles
    # within a row) when the scratch holds at least one row
    tiles_x = -(-state.f1.width // _lib.TILE_W)
    r = state.scratch_tiles
    if r >= tiles_x:
        r = r // tiles_x * tiles_x
    f2s = _lib.ptr_array([state.pyramid.levels[l].values for l in range(state.spec.levels)])
    full = state.desc
    try:
        for t0 in range(0, state.n_tiles, r):
            d = _lib.PartialDesc()
            _lib.C.pointer(d)[0] = full
            d.tile_begin, d.tile_end = t0, min(t0 + r, state.n_tiles)
            state.desc = d
            caches = (_lib.C.c_void_p * len(state.levels))(
                *[lv.cache.data_ptr() - 4 * t0 * pt for lv, pt in zip(state.levels, per_tile)])
            _contract(state, centroids, flags, f2s, caches)
            _gather(state, centroids, flags, f2s, caches, out)
    finally:
        state.desc = full


def _sample_tile_mode(state: SparseVolumeState, centroids: CentroidField,
                      out: torch.Tensor) -> None:
    """Contract then gather.  On the tensor-core path the frame is cut into
    tile ranges and gather(range i) runs on a side stream while contract(range
    i+1) runs on the caller's stream: the memory-bound sampler overlaps the
    latency-bound contraction.  gather(range) depends only on contract(range)
    of the same iteration; the caller's stream joins the side stream at the
    end, so the next iteration's contraction never races this one's gather."""
    flags = coords_flags(centroids, state.strict)
    if not state.cache_enabled:
        flags |= _lib.CVB_NO_CACHE
    if state.scratch_tiles:
        _sample_scratch_ranges(state, centroids, flags, out)
        return
    f2s, caches = _contract_args(state, centroids, flags)
    splits = state.pipeline_splits
    if splits <= 1:
        _contract(state, centroids, flags, f2s, caches)
        _gather(state, centroids, flags, f2s, caches, out)
        return
    main = torch.cuda.current_stream(state.device)
    if state._side_stream is None:
        state._side_stream = torch.cuda.Stream(state.device)
    side = state._side_stream
    out.record_stream(side)
    centroids.coords.record_stream(side)
    full = state.desc
    try:
        for d in _range_descs(state, splits):
            state.desc = d
            _contract(state, centroids, flags, f2s, caches)
            ev = torch.cuda.Event()
            ev.record(main)
            side.wait_event(ev)
            with torch.cuda.stream(side):
                _gather(state, centroids, flags, f2s, caches, out)
    finally:
        state.desc = full
    ev = torch.cuda.Event()
    ev.record(side)
    main.wait_event(ev)


@on_device
def sample_iteration(state: SparseVolumeState, centroids: CentroidField,
                     out: Optional[torch.Tensor] = None) -> CostMaps:
    """One lookup iteration (sparse.py:411-452); returns [H, W, L, 2r+1, 2r+1]."""
    _check_grid(state, centroids)
    f1, spec = state.f1, state.spec
    k1 = spec.window
    if out is None:
        out = torch.empty((f1.height, f1.width, spec.levels, k1, k1), dtype=torch.float32,
                          device=state.device)
    if state.mode == "tile":
        _sample_tile_mode(state, centroids, out)
        if state.ref_counters:
            _accumulate_ref_counters(state, centroids)
    else:
        _sample_block_mode(state, centroids, out)
    state.iteration += 1
    return CostMaps(values=out, radius=spec.radius)


@on_device
def sample_iteration_raft(state: SparseVolumeState, centroids: CentroidField,
                          out: torch.Tensor) -> torch.Tensor:
    """One lookup iteration written straight into RAFT's CorrBlock layout:
    out [L * (2r+1)^2, H, W], window index dx * (2r+1) + dy (the order RAFT's
    meshgrid(dy, dx) delta produces), by the sampler kernel itself
    (CVB_OUT_RAFT; fast r=4 tile path)."""
    if state.mode != "tile" or state.strict or state.spec.radius != 4:
        raise ValueError("CVB_OUT_RAFT needs a fast-arithmetic r=4 tile-mode state")
    _check_grid(state, centroids)
    spec, f1 = state.spec, state.f1
    if out.shape != (spec.levels * spec.window ** 2, f1.height, f1.width) or \
            out.dtype != torch.float32 or not out.is_contiguous():
        raise ValueError("out must be a contiguous float32 [L*(2r+1)^2, H, W] tensor")
    flags = coords_flags(centroids, False)
    if not state.cache_enabled:
        flags |= _lib.CVB_NO_CACHE
    f2s, caches = _contract_args(state, centroids, flags)
    _contract(state, centroids, flags, f2s, caches)
    _gather(state, centroids, flags | _lib.CVB_OUT_RAFT, f2s, caches, out)
    state.iteration += 1
    return out


def memory_footprint(state: SparseVolumeState) -> Dict:
    """Byte accounting of the sampler state (sparse.py:455-496).

    Same keys as the reference.  total_bytes = mask + capacity + features,
    where features are the source map plus the pyramid levels (the GPU keeps
    them row-major; no patch-major copy), capacity is the tile cache (tile
    mode) or the block-store arena (block mode), and mask is the bit-packed
    block mask (block mode) or the tile metadata (tile mode).
    """
    per_level = []
    mask_total = used_total = cap_total = blocks_used_total = 0
    feat_total = state.f1.values.numel() * 4
    for lvl, lv in enumerate(state.levels):
        fbytes = state.pyramid.levels[lvl].values.numel() * 4 if lvl > 0 else 0
        if state.mode == "block":
            mask_bytes = (lv.block_positions + 7) // 8
            block_bytes = lv.store.used_bytes()
            cap_bytes = lv.store.capacity_bytes()
            blocks_used = lv.store.used
        else:
            mask_bytes = state.meta.numel() * 4 // len(state.levels)
            cap_bytes = lv.cache.numel() * 4
            block_bytes = cap_bytes
            blocks_used = 0
        fbytes_all = state.pyramid.levels[lvl].values.numel() * 4
        per_level.append({"level": lvl, "mask_bytes": mask_bytes, "block_bytes": block_bytes,
                          "capacity_bytes": cap_bytes, "feature_bytes": fbytes_all,
                          "blocks_used": blocks_used,
                          "block_positions": lv.block_positions})
        mask_total += mask_bytes
        used_total += block_bytes
        cap_total += cap_bytes
        feat_total += fbytes
        blocks_used_total += blocks_used
    feat_total += state.pyramid.levels[0].values.numel() * 4
    # tensor-core path: the fp16 hi/lo operand planes of F1 and of every level
    split_total = 0
    if state.tc:
        split_total = state.tc_f1.numel() + sum(t.numel() for t in state.tc_f2)
    return {"levels": per_level, "mask_bytes": mask_total, "block_bytes": used_total,
            "capacity_bytes": cap_total, "feature_bytes": feat_total,
            "split_bytes": split_total, "blocks_used": blocks_used_total,
            "total_bytes": mask_total + cap_total + feat_total + split_total}


@on_device
def sample_iteration_timed(state: SparseVolumeState, centroids: CentroidField,
                           out: torch.Tensor) -> Tuple[torch.cuda.Event, ...]:
    """Tile-mode iteration with CUDA events around each kernel (bench helper).

    Returns (e0, e1, e2): contraction = e0->e1, gather/sampler = e1->e2,
    recorded on the launching (current) stream.
    """
    if state.mode != "tile":
        raise ValueError("timed iterations need a tile-mode state")
    _check_grid(state, centroids)
    flags = coords_flags(centroids, state.strict)
    if not state.cache_enabled:
        flags |= _lib.CVB_NO_CACHE
    f2s, caches = _contract_args(state, centroids, flags)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    _contract(state, centroids, flags, f2s, caches)
    ev[1].record()
    _gather(state, centroids, flags, f2s, caches, out)
    ev[2].record()
    state.iteration += 1
    return tuple(ev)
