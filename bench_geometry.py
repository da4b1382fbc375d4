"""Independent CPU geometry routine for the roofline's algorithmic work.

For a workload (seeded synthetic scenario, fp32-quantised centroids) it counts,
per iteration t, the compulsory cost cells any caching sampler must compute:
the first touch of each (query, level, cell) over the (2r+2)^2 supports
clipped to the level grid, i.e. |W_t(q) \\ U_{s<t} W_s(q)|.  flops_alg per
iteration = 2*D*first_touch_t.  Also the window-cell totals (what on-demand
evaluates).  Never uses the kernels under test.  Writes profiles/geometry_<cfg>.json.

    python bench_geometry.py C4
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2505_16942_b200.scenario import gen_scenario  # noqa: E402
from paper_2505_16942_b200.types import LookupSpec  # noqa: E402

CONFIGS = {
    "C1": (46, 62, 256, 4, 4, 12, False),
    "C2": (135, 240, 256, 4, 4, 32, False),
    "C3": (270, 480, 256, 4, 4, 12, True),
    "C4": (540, 960, 256, 4, 4, 12, False),
}


def first_touch(coords_list, level, radius, th, tw, chunk=8192):
    n_iter = len(coords_list)
    p = coords_list[0].shape[0] * coords_list[0].shape[1]
    offs = np.arange(-radius, radius + 2, dtype=np.int64)
    s = offs.size
    hist = np.zeros(n_iter, dtype=np.int64)
    window = np.zeros(n_iter, dtype=np.int64)
    flat = [c.reshape(-1, 2).astype(np.float64) for c in coords_list]
    for q0 in range(0, p, chunk):
        q1 = min(p, q0 + chunk)
        nq = q1 - q0
        keys = []
        for t, c in enumerate(flat):
            x0 = np.floor(c[q0:q1, 0] / 2.0 ** level).astype(np.int64)
            y0 = np.floor(c[q0:q1, 1] / 2.0 ** level).astype(np.int64)
            ty = (y0[:, None] + offs[None, :])[:, :, None]
            tx = (x0[:, None] + offs[None, :])[:, None, :]
            valid = (ty >= 0) & (ty < th) & (tx >= 0) & (tx < tw)
            q = np.broadcast_to(np.arange(nq)[:, None, None], (nq, s, s))
            cell = np.broadcast_to(ty * tw + tx, (nq, s, s))
            k = (q[valid] * (th * tw) + cell[valid]) * 64 + t
            window[t] += k.size
            keys.append(k)
        k = np.sort(np.concatenate(keys))
        cellkey = k >> 6
        start = np.ones(k.size, dtype=bool)
        start[1:] = cellkey[1:] != cellkey[:-1]
        hist += np.bincount((k[start] & 63), minlength=n_iter)[:n_iter]
    return hist, window


def main(name: str) -> None:
    h, w, d, r, levels, n_iter, normalize = CONFIGS[name]
    t0 = time.time()
    sc = gen_scenario(0, (h, w, d), n_iter, LookupSpec(r, levels, normalize),
                      coords_dtype=np.float32)
    per_level = []
    first = np.zeros(n_iter, dtype=np.int64)
    windows = np.zeros(n_iter, dtype=np.int64)
    th, tw = h, w
    for lvl in range(levels):
        ft, win = first_touch(sc.centroid_fields, lvl, r, th, tw)
        per_level.append({"level": lvl, "grid": [th, tw], "first_touch": ft.tolist(),
                          "window_cells": win.tolist()})
        first += ft
        windows += win
        th, tw = th // 2, tw // 2
        print(f"{name} level {lvl}: union {int(ft.sum())} ({time.time() - t0:.0f}s)",
              flush=True)
    out = {
        "config": name, "dims": [h, w, d], "radius": r, "levels": levels,
        "iterations": n_iter, "seed": 0, "coords": "float32",
        "first_touch_per_iter": first.tolist(),
        "window_cells_per_iter": windows.tolist(),
        "union_cells": int(first.sum()),
        "flops_alg_per_iter": [2 * d * int(v) for v in first],
        "flops_alg_run": 2 * d * int(first.sum()),
        "levels_detail": per_level,
    }
    path = ROOT / "profiles" / f"geometry_{name}.json"
    path.parent.mkdir(exist_ok=True)
    path.write_text(json.dumps(out, indent=1))
    print(f"wrote {path}: union {out['union_cells']}, flops_alg {out['flops_alg_run'] / 1e9:.1f} GF")


if __name__ == "__main__":
    for cfg in sys.argv[1:] or ["C4"]:
        main(cfg)
