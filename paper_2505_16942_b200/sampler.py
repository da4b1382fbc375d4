"""CorrSampler: the per-iteration `__call__(coords)` lookup with a variant switch.

The reference has no class API (its harness calls the three samplers
directly, harness.py:36,190-274,459-471); RAFT/SEA-RAFT callers use a
`CorrBlock(fmap1, fmap2)(coords)` object.  CorrSampler provides that shape on
top of the reference-named functions:

    sampler = CorrSampler(fmap1, fmap2, LookupSpec(4, 4), variant="partial")
    for it in range(iters):
        costs = sampler(coords)          # [H, W, L, 2r+1, 2r+1] on the GPU

variant: "partial" (sparse.py, the north-star path: incremental tile cache),
"ondemand" (no state across iterations: fast arithmetic recomputes every
query tile's window union on tcgen05 each iteration into a bounded scratch;
strict runs the reference's per-query dots, ondemand.py), "dense" (dense.py:
the all-pairs volume, on tcgen05 unless strict; raises MemoryError when the
volume would not fit, the analogue of the reference bench's oom row,
harness.py:330-333).
"""

from __future__ import annotations

from typing import Optional

import torch

from .dense import build_feature_pyramid, build_volume_pyramid, estimate_dense_bytes, lookup_dense
from .ondemand import lookup_on_demand
from .sparse import init_state, init_state_batch, memory_footprint, sample_iteration
from .types import CentroidField, CostMaps, FeatureMap, LookupSpec

VARIANTS = ("dense", "ondemand", "partial")
#: tiles per scratch range of the fast on-demand variant (8 per B200 SM)
ONDEMAND_SCRATCH_TILES = 8 * 148
_ALIASES = {"sparse": "partial"}


class CorrSampler:
    def __init__(self, fmap1, fmap2, spec: LookupSpec, variant: str = "partial", block: int = 8,
                 cache: bool = True, strict: bool = False, mode: str = "tile",
                 dense_mode: str = "pool_features", dense_limit_bytes: Optional[int] = None,
                 check: bool = True, graph: bool = False, **state_kwargs):
        variant = _ALIASES.get(variant, variant)
        if variant not in VARIANTS:
            raise ValueError(f"variant must be one of {VARIANTS}, got {variant!r}")
        self.variant = variant
        self.spec = spec
        self.strict = strict
        self.f1 = fmap1 if isinstance(fmap1, FeatureMap) else FeatureMap(fmap1, check=check)
        self.f2 = fmap2 if isinstance(fmap2, FeatureMap) else FeatureMap(fmap2, check=check)
        self.check = check
        # graph=True (partial variant): after one eager call, each iteration's
        # launch sequence (tiler, contraction, sampler) is replayed from a
        # captured CUDA graph on static coordinate / output buffers — for
        # launch-bound frames; the returned tensor is reused by the next call
        if graph and (variant != "partial" or mode != "tile"):
            # block mode sizes its store on the host (.item() syncs, host-side
            # growth): nothing a replayed graph could reproduce
            raise ValueError("graph=True needs variant='partial' with mode='tile'")
        self.graph = graph
        self._graph = None
        self._g_coords = None
        self._g_out = None
        self._eager_calls = 0
        self.state = None
        self.volume = None
        self.pyramid = None
        if variant == "partial":
            self.state = init_state(self.f1, self.f2, spec, block, cache_enabled=cache,
                                    mode=mode, strict=strict, **state_kwargs)
            self.pyramid = self.state.pyramid
        elif variant == "ondemand":
            if not strict and self.f1.dims <= 256 and spec.radius <= 8:
                # fast on-demand: every iteration recomputes each query tile's
                # window union on tcgen05 into a bounded scratch (ranges of
                # ONDEMAND_SCRATCH_TILES tiles) and samples it; nothing is kept
                # across iterations (no incremental cache)
                self.state = init_state(self.f1, self.f2, spec, block, cache_enabled=False,
                                        mode="tile", scratch_tiles=ONDEMAND_SCRATCH_TILES)
                self.pyramid = self.state.pyramid
            else:  # reference arithmetic: per-query window cells, FFMA-free dots
                self.pyramid = build_feature_pyramid(self.f2, spec.levels)
        else:
            need = estimate_dense_bytes((self.f1.height, self.f1.width),
                                        (self.f2.height, self.f2.width), spec.levels)
            limit = dense_limit_bytes
            if limit is None:
                free, _ = torch.cuda.mem_get_info(self.f1.values.device)
                limit = int(free * 0.9)
            if need > limit:
                raise MemoryError(f"dense volume needs {need} bytes (> limit {limit})")
            self.volume = build_volume_pyramid(self.f1, self.f2, spec.levels, mode=dense_mode,
                                               strict=strict)

    def __call__(self, coords, out: Optional[torch.Tensor] = None) -> CostMaps:
        cents = coords if isinstance(coords, CentroidField) else CentroidField(coords,
                                                                                check=self.check)
        if self.variant == "partial":
            if self.graph:
                return self._graphed(cents, out)
            return sample_iteration(self.state, cents, out=out)
        if self.variant == "ondemand":
            if self.state is not None:
                return sample_iteration(self.state, cents, out=out)
            return lookup_on_demand(self.f1, self.pyramid, cents, self.spec, strict=self.strict,
                                    out=out)
        return lookup_dense(self.volume, cents, self.spec, strict=self.strict, out=out)

    def _graphed(self, cents: CentroidField, out: Optional[torch.Tensor]) -> CostMaps:
        c = cents.coords
        if self._graph is None:
            if self._eager_calls == 0:  # first call eagerly: library setup, iteration 0
                self._eager_calls += 1
                return sample_iteration(self.state, cents, out=out)
            self._g_coords = torch.empty_like(c)
            self._g_coords.copy_(c)
            k = self.spec.window
            self._g_out = torch.empty((self.f1.height, self.f1.width, self.spec.levels, k, k),
                                      dtype=torch.float32, device=c.device)
            g_cents = CentroidField(self._g_coords, check=False)
            torch.cuda.synchronize(c.device)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                sample_iteration(self.state, g_cents, out=self._g_out)
            self.state.iteration -= 1  # capture recorded the launches without running them
            self._graph = graph
        elif c.shape != self._g_coords.shape or c.dtype != self._g_coords.dtype:
            raise ValueError("graph mode needs coords of the captured shape and dtype")
        else:
            self._g_coords.copy_(c)
        self._graph.replay()
        self.state.iteration += 1
        res = self._g_out
        if out is not None:
            out.copy_(res)
            res = out
        return CostMaps(values=res, radius=self.spec.radius)

    def memory_bytes(self) -> int:
        """Analytic bytes the variant holds between iterations."""
        feats = self.f1.values.numel() * 4
        if self.state is not None:
            return memory_footprint(self.state)["total_bytes"]
        feats += sum(l.values.numel() * 4 for l in self.pyramid.levels) if self.pyramid else 0
        if self.variant == "dense":
            return self.volume.nbytes() + self.f1.values.numel() * 4 + \
                self.f2.values.numel() * 4
        return feats


class BatchCorrSampler:
    """A batch of independent image pairs (C5: batched 4K sweep).

    fmaps1 / fmaps2: [B, H, W, D]; `__call__(coords [B, H, W, 2])` returns
    [B, H, W, L, 2r+1, 2r+1].  The partial variant keeps ONE tile-mode state
    for all pairs (`sparse.init_state_batch`): each iteration is one plan,
    one contraction and one sampler launch over every pair's tiles, and with
    graph=True (default) the iteration is replayed from a captured CUDA graph.
    Per pair the costs are bit-identical to a single-pair CorrSampler.  Pairs
    shard across ranks with no data-path collective (`parallel.batch_slices`);
    `parallel.gather_bands` all-gathers the per-rank slices when every rank
    needs every pair's costs.  The reference has no batching.
    The dense / on-demand variants run pair by pair.
    """

    def __init__(self, fmaps1: torch.Tensor, fmaps2: torch.Tensor, spec: LookupSpec,
                 variant: str = "partial", strict: bool = False, cache: bool = True,
                 graph: bool = True, **kwargs):
        if fmaps1.dim() != 4 or fmaps1.shape != fmaps2.shape:
            raise ValueError("fmaps must both be [B, H, W, D] with equal shapes")
        variant = _ALIASES.get(variant, variant)
        self.spec = spec
        self.variant = variant
        self.batch, self.height, self.width = fmaps1.shape[:3]
        self.state = None
        self.samplers = []
        self.graph = graph and variant == "partial"
        self._graph = None
        self._g_coords = None
        self._g_out = None
        self._own_out = None
        self._calls = 0
        if variant == "partial":
            self.state = init_state_batch(fmaps1, fmaps2, spec, strict=strict,
                                          cache_enabled=cache, **kwargs)
        else:
            self.samplers = [CorrSampler(FeatureMap(fmaps1[b], check=False),
                                         FeatureMap(fmaps2[b], check=False), spec,
                                         variant=variant, strict=strict, cache=cache,
                                         check=False, **kwargs)
                             for b in range(fmaps1.shape[0])]

    def __len__(self) -> int:
        return self.batch

    def states(self):
        """The partial-sampler state(s): one batched state (device counters,
        footprint)."""
        return [self.state] if self.state is not None else [s.state for s in self.samplers]

    def _out_shape(self):
        k = self.spec.window
        return (self.batch, self.height, self.width, self.spec.levels, k, k)

    def __call__(self, coords: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        b, h, w = coords.shape[:3]
        if (b, h, w) != (self.batch, self.height, self.width):
            raise ValueError(f"coords {tuple(coords.shape)} do not match the batch "
                             f"[{self.batch}, {self.height}, {self.width}, 2]")
        if out is None:
            if self.graph and self.state is not None:
                # graph mode: one persistent result buffer, reused by the next call
                if self._own_out is None:
                    self._own_out = torch.empty(self._out_shape(), dtype=torch.float32,
                                                device=coords.device)
                out = self._own_out
            else:
                out = torch.empty(self._out_shape(), dtype=torch.float32, device=coords.device)
        if self.state is None:
            for i, s in enumerate(self.samplers):
                s(CentroidField(coords[i], check=False), out=out[i])
            return out
        flat = coords.reshape(b * h, w, 2)
        view = out.view(b * h, w, *out.shape[3:])
        if not self.graph or self._calls == 0:  # eager (the first call sets up, iteration 0)
            self._calls += 1
            sample_iteration(self.state, CentroidField(flat, check=False), out=view)
            return out
        # one captured iteration per output buffer: callers that reuse `out`
        # (the usual loop) replay it with no extra copy of the cost maps
        if self._graph is None or self._g_out != out.data_ptr() or \
                flat.dtype != self._g_coords.dtype:
            self._g_coords = torch.empty_like(flat)
            self._g_coords.copy_(flat)
            g_cents = CentroidField(self._g_coords, check=False)
            torch.cuda.synchronize(flat.device)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                sample_iteration(self.state, g_cents, out=view)
            self.state.iteration -= 1  # capture recorded the launches without running them
            self._graph, self._g_out = graph, out.data_ptr()
        else:
            self._g_coords.copy_(flat)
        self._graph.replay()
        self.state.iteration += 1
        self._calls += 1
        return out
