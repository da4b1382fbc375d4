"""GPU access recorder and block occupancy.

The reference's analyzer (analyzer.py:31-116) logs every (source, target)
cell reached with nonzero bilinear weight over a scenario's iterations and
reports the percentage of B^2 x B^2 blocks of the level volume that contain a
touched cell, for the row-major and patch-major layouts — the paper's Suppl.
Table 1 study.  The reference materialises the log as
int64 codes (hundreds of millions at 8K); here the kernels keep only what the
study needs: the touched-cell count (per query, cells not covered by an
earlier window of the same query) and one bitmask of touched block positions
per (block size, layout).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

import torch

from . import _lib
from ._backend import on_device, stream_handle
from .dense import coords_flags, pooled_dims
from .types import CentroidField, LookupSpec

LAYOUTS = ("row-major", "patch-major")


@dataclass
class LevelAccess:
    level: int
    src_shape: Tuple[int, int]
    tgt_shape: Tuple[int, int]
    first_touch: List[int]                 # touched cells first reached per iteration
    occupancy: Dict[Tuple[int, str], float] = field(default_factory=dict)

    @property
    def touched_cells(self) -> int:
        """Size of the reference AccessLog of this level."""
        return sum(self.first_touch)


def _groups(shape: Tuple[int, int], block: int, layout: str) -> int:
    h, w = shape
    if layout == "row-major":
        return -(-(h * w) // (block * block))
    if layout == "patch-major":
        return -(-h // block) * -(-w // block)
    raise ValueError(f"layout must be one of {LAYOUTS}, got {layout!r}")


@on_device
def record_occupancy(centroid_fields: Sequence[CentroidField], spec: LookupSpec,
                     tgt_shape: Tuple[int, int], block_sizes: Sequence[int] = (1, 2, 4, 8),
                     layouts: Sequence[str] = LAYOUTS, trim: bool = True) -> List[LevelAccess]:
    """Touched cells and block occupancy per level over a centroid sequence
    (record_run + occupancy, analyzer.py:31-113).  trim=False counts the full
    (2r+2)^2 support (the sampler's compulsory cells)."""
    cents = list(centroid_fields)
    if not cents or len(cents) > 64:
        raise ValueError("1..64 centroid fields")
    h1, w1 = cents[0].height, cents[0].width
    dev = cents[0].coords.device
    flags = coords_flags(cents[0], False) | (0 if trim else _lib.CVB_ACCESS_NO_TRIM)
    ptrs = _lib.ptr_array([c.coords for c in cents])
    out = []
    for lvl in range(spec.levels):
        th, tw = pooled_dims(tgt_shape, lvl)
        ft = torch.zeros(len(cents), dtype=torch.int64, device=dev)
        _lib.call("cvb_access_union", ptrs, len(cents), h1, w1, lvl, spec.radius, th, tw, flags,
                  _lib.ptr(ft), stream_handle())
        acc = LevelAccess(lvl, (h1, w1), (th, tw), [int(v) for v in ft.tolist()])
        for b in block_sizes:
            if b < 1:
                raise ValueError("block must be >= 1")
            for layout in (LAYOUTS if b == 1 else layouts):
                n_gs, n_gt = _groups((h1, w1), b, layout), _groups((th, tw), b, layout)
                if b == 1:
                    # layouts only permute cells: occupancy = touched / positions
                    acc.occupancy[(1, layout)] = 100.0 * acc.touched_cells / (n_gs * n_gt)
                    continue
                wpr = (n_gt + 31) // 32
                mask = torch.zeros((n_gs, wpr), dtype=torch.int32, device=dev)
                for c in cents:
                    _lib.call("cvb_access_blocks", _lib.ptr(c.coords), h1, w1, lvl, spec.radius,
                              th, tw, b, int(layout == "patch-major"), flags, _lib.ptr(mask), wpr,
                              stream_handle())
                lut = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int64,
                                   device=dev)
                touched = int(lut[mask.view(torch.uint8).long()].sum().item())
                acc.occupancy[(b, layout)] = 100.0 * touched / (n_gs * n_gt)
        out.append(acc)
    return out
