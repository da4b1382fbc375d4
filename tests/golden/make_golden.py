"""Generates tests/golden/golden.npz by running the REFERENCE itself.

Run in the build container (needs the reference package: oracle/_ref built by
oracle/build.sh, or /root/reference/pkg/src on sys.path):

    python tests/golden/make_golden.py

Every array is produced by corrvol 0.1.0's own public functions (cython lane
when available — bit-identical to its numpy lane, test_backends.py:70-90).
The fixtures pin both the CPU oracle (tests/test_oracle.py) and the CUDA path
(tests/test_gpu_parity.py) without needing the reference at run time.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import import_reference  # noqa: E402

cv = import_reference()
if cv is None:
    sys.path.insert(0, "/root/reference/pkg/src")
    import corrvol as cv  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden.npz"
G = {}


def fmap(h, w, d, seed):
    rng = np.random.default_rng(seed)
    return cv.FeatureMap(values=rng.standard_normal((h, w, d)).astype(np.float32))


def cents(h, w, seed, spread=3.0):
    rng = np.random.default_rng(seed)
    ys, xs = np.mgrid[0:h, 0:w]
    c = np.stack([xs, ys], axis=-1).astype(np.float64)
    c += rng.uniform(-spread, spread, size=c.shape)
    return cv.CentroidField(coords=c)


def lookup_case(name, f1, f2, spec, fields, blocks=(1, 4), cache=True):
    """All reference samplers on the same inputs."""
    G[f"{name}/f1"] = f1.values
    G[f"{name}/f2"] = f2.values
    G[f"{name}/spec"] = np.array([spec.radius, spec.levels, int(spec.normalize)])
    G[f"{name}/n_iter"] = np.array(len(fields))
    pyr = cv.build_feature_pyramid(f2, spec.levels)
    vol_pf = cv.build_volume_pyramid(f1, f2, spec.levels, mode="pool_features")
    vol_pv = cv.build_volume_pyramid(f1, f2, spec.levels, mode="pool_volume")
    states = {b: cv.init_state(f1, f2, spec, b, cache_enabled=cache) for b in blocks}
    for it, c in enumerate(fields):
        G[f"{name}/coords{it}"] = c.coords
        od = cv.lookup_on_demand(f1, pyr, c, spec).values
        G[f"{name}/out{it}"] = od
        if it == 0:
            G[f"{name}/dense_pv{it}"] = cv.lookup_dense(vol_pv, c, spec).values
        assert np.array_equal(cv.lookup_dense(vol_pf, c, spec).values, od)
        for b, st in states.items():
            sp = cv.sample_iteration(st, c).values
            assert np.array_equal(sp, od), (name, b)
            G[f"{name}/B{b}/blocks{it}"] = np.array(st.counter.blocks_computed)
            G[f"{name}/B{b}/used{it}"] = np.array([lv.store.used for lv in st.levels])
            G[f"{name}/B{b}/union{it}"] = np.array([int(lv.mask_union.sum()) for lv in st.levels])
    for b, st in states.items():
        fp = cv.memory_footprint(st)
        G[f"{name}/B{b}/footprint"] = np.array(
            [fp["mask_bytes"], fp["block_bytes"], fp["capacity_bytes"], fp["blocks_used"]])
        for lvl, lv in enumerate(st.levels):
            flat = lv.block_ids.ravel()
            nz = np.flatnonzero(flat >= 0)
            G[f"{name}/B{b}/ids_l{lvl}"] = np.stack([nz, flat[nz]]).astype(np.int32)
            G[f"{name}/B{b}/shape_l{lvl}"] = np.array(lv.block_ids.shape)
    for lvl in range(spec.levels):
        G[f"{name}/pv_mat{lvl}"] = vol_pv.level_mats[lvl] if vol_pv.level_mats[lvl].size <= 20000 \
            else np.zeros(0, np.float32)
    counter = cv.WorkCounter()
    for c in fields:
        cv.lookup_on_demand(f1, pyr, c, spec, counter=counter)
    G[f"{name}/od_dots"] = np.array(counter.dot_products)


def main():
    # pyramid (test_dense.py:59-65) incl. odd dims
    f2 = fmap(9, 7, 3, 4)
    pyr = cv.build_feature_pyramid(f2, 3)
    G["pyr/f2"] = f2.values
    for lvl in range(3):
        G[f"pyr/l{lvl}"] = pyr.levels[lvl].values
    f2b = fmap(10, 12, 8, 5)
    pyrb = cv.build_feature_pyramid(f2b, 3)
    G["pyr8/f2"] = f2b.values
    for lvl in range(3):
        G[f"pyr8/l{lvl}"] = pyrb.levels[lvl].values

    # floors (sparse.py:251-259) on awkward coordinates
    xs = np.array([0.0, 1.0, -1.0, 0.5, -0.5, 2.999999999, -2.000000001, 1e-300, -1e-300,
                   12345.678, -9876.5, 7.0 + 2 ** -30, 3.75, 1e9 + 0.5, -3.0],
                  dtype=np.float64)
    coords = np.stack(np.meshgrid(xs, xs[::-1]), axis=-1).reshape(len(xs), len(xs), 2)
    G["floors/coords"] = coords
    st = cv.init_state(fmap(len(xs), len(xs), 2, 1), fmap(4, 4, 2, 2), cv.LookupSpec(1, 1), 2)
    for lvl in range(4):
        x0, y0, fx, fy = cv.sparse._level_centroid_floors(st, cv.CentroidField(coords=coords),
                                                          lvl)
        G[f"floors/x0_{lvl}"], G[f"floors/y0_{lvl}"] = x0, y0
        G[f"floors/fx_{lvl}"], G[f"floors/fy_{lvl}"] = fx, fy

    # bilinear known answers (test_types.py:130-154)
    grid = np.array([[1.0, 2.0], [3.0, 4.0]], dtype=np.float32)
    pts = np.array([[0, 0], [0.5, 0], [0.5, 0.5], [-0.5, 0], [1, 1], [1.5, 1.5], [-1, -1],
                    [0.25, 0.75], [0.999, 0.001]], dtype=np.float64)
    G["bilinear/grid"] = grid
    G["bilinear/pts"] = pts
    G["bilinear/vals"] = np.array([cv.types.bilinear_tap(grid, x, y) for x, y in pts])

    # kernel lane (test_backends.py)
    rng = np.random.default_rng(8)
    a = rng.standard_normal((23, 17)).astype(np.float32)
    b = rng.standard_normal((19, 17)).astype(np.float32)
    k = cv._backend.get_kernels()
    G["lane/a"], G["lane/b"], G["lane/pairs"] = a, b, k.corr_pairs(a, b)
    f1g = rng.standard_normal((31, 13)).astype(np.float32)
    f2g = rng.standard_normal((40, 13)).astype(np.float32)
    idx = rng.integers(0, 40, size=31).astype(np.int64)
    valid = (rng.random(31) < 0.7).astype(np.uint8)
    G["lane/g_f1"], G["lane/g_f2"], G["lane/g_idx"], G["lane/g_valid"] = f1g, f2g, idx, valid
    G["lane/gather"] = k.corr_gather(f1g, f2g, idx, valid)
    at = rng.standard_normal((11, 16, 24)).astype(np.float32)
    bt = rng.standard_normal((11, 9, 24)).astype(np.float32)
    G["lane/at"], G["lane/bt"], G["lane/mmm"] = at, bt, k.block_mmm(at, bt)

    # samplers
    lookup_case("small", fmap(7, 9, 5, 0), fmap(7, 9, 5, 1), cv.LookupSpec(2, 2),
                [cents(7, 9, 2), cents(7, 9, 3)], blocks=(1, 2, 3, 4, 5, 8))
    lookup_case("norm", fmap(5, 5, 4, 4), fmap(5, 5, 4, 5), cv.LookupSpec(1, 1, True),
                [cents(5, 5, 6)], blocks=(2,))
    # every window outside the grid: the reference's sparse path raises
    # IndexError here (empty store indexed, sparse.py:373-374); dense and
    # on-demand return zeros, which is what the B200 partial path returns.
    lookup_case("oob", fmap(4, 4, 3, 13), fmap(4, 4, 3, 14), cv.LookupSpec(1, 1),
                [cv.CentroidField(coords=np.full((4, 4, 2), 100.0))], blocks=())
    ys, xs_ = np.mgrid[0:3, 0:3]
    lookup_case("intr0", fmap(3, 3, 2, 15), fmap(3, 3, 2, 16), cv.LookupSpec(0, 1),
                [cv.CentroidField(coords=np.stack([xs_, ys], -1).astype(np.float64))],
                blocks=(1, 2))
    # padded-grid semantics probe: window wholly outside
    # the 10x10 grid but inside the 16x16 padded grid
    c = np.full((10, 10, 2), -50.0)
    c[0, 0] = (13.0, 13.0)
    lookup_case("padded", fmap(10, 10, 4, 21), fmap(10, 10, 4, 22), cv.LookupSpec(1, 1),
                [cv.CentroidField(coords=c)], blocks=(8,))
    sc = cv.gen_scenario(1003, (20, 16, 32), 4, cv.LookupSpec(4, 3))
    lookup_case("scen", sc.f1, sc.f2, sc.spec, sc.centroid_fields, blocks=(1, 4, 8))
    sc2 = cv.gen_scenario(7, (12, 16, 256), 2, cv.LookupSpec(4, 2, True))
    lookup_case("d256", sc2.f1, sc2.f2, sc2.spec, sc2.centroid_fields, blocks=(8,))
    sc3 = cv.gen_scenario(11, (9, 13, 8), 3, cv.LookupSpec(2, 2))
    lookup_case("nocache", sc3.f1, sc3.f2, sc3.spec, sc3.centroid_fields, blocks=(2,),
                cache=False)

    # computation masks + incremental ids (sparse.py:262-309), per iteration & level
    sc4 = cv.gen_scenario(5, (17, 23, 4), 3, cv.LookupSpec(3, 3))
    st4 = cv.init_state(sc4.f1, sc4.f2, sc4.spec, 4)
    G["mask/spec"] = np.array([3, 3, 4, 17, 23])
    for it, cf in enumerate(sc4.centroid_fields):
        G[f"mask/coords{it}"] = cf.coords
        for lvl in range(3):
            m = cv.set_computation_mask(st4, cf, lvl)
            G[f"mask/m{it}_{lvl}"] = np.argwhere(m).astype(np.int32)
            pos, ids = cv.compute_block_indices(st4, m, lvl)
            G[f"mask/pos{it}_{lvl}"], G[f"mask/ids{it}_{lvl}"] = pos, ids
            cv.sampled_block_mmm(st4, lvl, pos)
    G["mask/n_src"] = np.array(st4.n_src_tiles)
    G["mask/n_tgt"] = np.array([lv.n_tgt_tiles for lv in st4.levels])

    np.savez_compressed(OUT, **G)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB, {len(G)} arrays)")


if __name__ == "__main__":
    main()
