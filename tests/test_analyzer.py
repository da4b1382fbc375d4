"""GPU access recorder / occupancy against the reference analyzer
(analyzer.py:31-116): identical touched-cell counts and occupancy percentages."""

import numpy as np
import pytest
import torch

import paper_2505_16942_b200 as cvb
from oracle import import_reference

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,dims,n,levels", [(0, (16, 24, 4), 5, 2), (3, (33, 29, 4), 8, 3),
                                                 (11, (64, 64, 4), 16, 1)])
def test_occupancy_matches_reference(cuda, seed, dims, n, levels):
    ref = import_reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from corrvol.analyzer import occupancy as ref_occ, record_run
    from corrvol.harness import gen_scenario as ref_gen

    spec = cvb.LookupSpec(4, levels)
    ours_sc = cvb.gen_scenario(seed, dims, n, spec)
    ref_sc = ref_gen(seed, dims, n, ref.LookupSpec(4, levels))
    logs = record_run(ref_sc)
    cents = [cvb.CentroidField(torch.from_numpy(c).to(cuda)) for c in ours_sc.centroid_fields]
    got = cvb.record_occupancy(cents, spec, dims[:2], block_sizes=(1, 2, 4, 8))
    for acc, log in zip(got, logs):
        assert acc.touched_cells == log.entries.size
        for (b, layout), pct in acc.occupancy.items():
            assert pct == ref_occ(log, b, layout), (acc.level, b, layout)


def test_untrimmed_union_is_the_compulsory_cell_count(cuda):
    """trim=False: per-level union of (2r+2)^2 supports clipped to the grid —
    the sampler's compulsory cells, checked by brute force."""
    spec = cvb.LookupSpec(4, 2)
    sc = cvb.gen_scenario(5, (20, 18, 4), 4, spec)
    cents = [cvb.CentroidField(torch.from_numpy(c).to(cuda)) for c in sc.centroid_fields]
    got = cvb.record_occupancy(cents, spec, (20, 18), block_sizes=(), trim=False)
    for lvl, acc in enumerate(got):
        th, tw = cvb.pooled_dims((20, 18), lvl)
        total = 0
        for y in range(20):
            for x in range(18):
                cells = set()
                for c in sc.centroid_fields:
                    x0 = int(np.floor(c[y, x, 0] / 2 ** lvl))
                    y0 = int(np.floor(c[y, x, 1] / 2 ** lvl))
                    for cy in range(y0 - 4, y0 + 6):
                        for cx in range(x0 - 4, x0 + 6):
                            if 0 <= cy < th and 0 <= cx < tw:
                                cells.add((cy, cx))
                total += len(cells)
        assert acc.touched_cells == total


@pytest.mark.parametrize("cfg", ["C1", "C4"])
def test_untrimmed_first_touch_matches_cpu_geometry(cuda, cfg):
    """The roofline's algorithmic work comes from the independent CPU routine
    (bench_geometry.py -> profiles/geometry_<cfg>.json); the GPU recorder
    reproduces its per-iteration first-touch counts exactly."""
    import json
    from pathlib import Path

    geom = json.loads((Path(__file__).resolve().parents[1] / "profiles" /
                       f"geometry_{cfg}.json").read_text())
    h, w, d = geom["dims"]
    spec = cvb.LookupSpec(geom["radius"], geom["levels"])
    sc = cvb.gen_scenario(geom["seed"], (h, w, d), geom["iterations"], spec,
                          coords_dtype=np.float32)
    cents = [cvb.CentroidField(torch.from_numpy(c).to(cuda)) for c in sc.centroid_fields]
    got = cvb.record_occupancy(cents, spec, (h, w), block_sizes=(), trim=False)
    per_iter = [sum(acc.first_touch[i] for acc in got) for i in range(geom["iterations"])]
    assert per_iter == geom["first_touch_per_iter"]
    assert sum(per_iter) == geom["union_cells"]
