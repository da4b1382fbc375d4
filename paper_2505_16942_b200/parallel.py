"""Multi-GPU sharding of the lookup: query-row bands (C4) and batch slices (C5).

Every output pixel depends only on F1[q], coords[q] and the full fmap2
pyramid, and the partial sampler's tile cache is per query tile, so a band
of query rows per rank is exact with no per-iteration exchange.  Bands start
at multiples of the 8-row query tile so every rank's tiles are whole tiles of
the full grid and results are bit-identical to the single-GPU run.
fmap2 (and hence its pyramid) is replicated; `gather_bands` is the optional
NCCL all-gather of the sampled costs.
"""

from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from ._lib import TILE_H


def row_bands(height: int, world: int, align: int = TILE_H) -> List[Tuple[int, int]]:
    """[start, stop) source-row band per rank; starts are multiples of `align`.

    Whole `align`-row units are dealt out as evenly as possible; ranks beyond
    the unit count get empty bands.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    units = (height + align - 1) // align
    base, extra = divmod(units, world)
    bands, u = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        start = min(u * align, height)
        stop = min((u + n) * align, height)
        bands.append((start, stop))
        u += n
    return bands


def batch_slices(batch: int, world: int) -> List[Tuple[int, int]]:
    """[start, stop) batch elements per rank (C5 batch sharding)."""
    base, extra = divmod(batch, world)
    out, s = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((s, s + n))
        s += n
    return out


def gather_bands(local: torch.Tensor, bands: Sequence[Tuple[int, int]],
                 group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """All-gather per-rank band outputs [rows_r, ...] into the full [H, ...].

    Bands may differ in size; each rank pads to the largest band so a single
    all_gather_into_tensor (NCCL ring/NVLS over NVLink) moves everything.
    """
    world = len(bands)
    rows = max(b - a for a, b in bands)
    tail = tuple(local.shape[1:])
    buf = torch.zeros((rows,) + tail, dtype=local.dtype, device=local.device)
    if local.shape[0]:
        buf[: local.shape[0]].copy_(local)
    if dist.get_backend(group) == "nccl":
        full = torch.empty((world * rows,) + tail, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(full, buf, group=group)
        chunks = [full[r * rows: (r + 1) * rows] for r in range(world)]
    else:  # gloo (CPU tests; ranks sharing one GPU): list all_gather on the host
        host = buf.cpu()
        chunks = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(chunks, host, group=group)
        chunks = [c.to(local.device) for c in chunks]
    parts = [chunks[r][: b - a] for r, (a, b) in enumerate(bands)]
    return torch.cat(parts, dim=0)
