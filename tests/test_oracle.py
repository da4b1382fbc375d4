"""Pins the CPU oracle to the reference: golden vectors (made by the reference
itself, tests/golden/make_golden.py) and, when oracle/_ref is built, live
random cases.  Everything compared with array_equal — the oracle restates the
reference arithmetic exactly."""

import numpy as np
import pytest

from oracle import corrvol_oracle as O

CASES = ["small", "norm", "oob", "intr0", "padded", "scen", "d256", "nocache"]


def _spec(g, name):
    r, l, n = (int(v) for v in g[f"{name}/spec"])
    return r, l, bool(n)


def test_pyramid_matches_golden(golden):
    for key in ("pyr", "pyr8"):
        levels = O.pyramid(golden[f"{key}/f2"], 3)
        for lvl in range(3):
            assert np.array_equal(levels[lvl], golden[f"{key}/l{lvl}"])


def test_floors_match_golden(golden):
    c = golden["floors/coords"]
    for lvl in range(4):
        x0, y0, fx, fy = O.level_floors(c, lvl)
        assert np.array_equal(x0, golden[f"floors/x0_{lvl}"])
        assert np.array_equal(y0, golden[f"floors/y0_{lvl}"])
        assert np.array_equal(fx, golden[f"floors/fx_{lvl}"])
        assert np.array_equal(fy, golden[f"floors/fy_{lvl}"])


def test_bilinear_known_answers(golden):
    grid = golden["bilinear/grid"]
    vals = [O.bilinear_tap(grid, x, y) for x, y in golden["bilinear/pts"]]
    assert np.array_equal(np.array(vals), golden["bilinear/vals"])
    # SPEC.md:71-73 known answers
    assert O.bilinear_tap(grid, 0.0, 0.0) == 1.0
    assert O.bilinear_tap(grid, 0.5, 0.0) == 1.5
    assert O.bilinear_tap(grid, -0.5, 0.0) == 0.5


def test_lane_dots_match_golden(golden):
    assert np.array_equal(O.corr_pairs(golden["lane/a"], golden["lane/b"]), golden["lane/pairs"])
    f1, f2 = golden["lane/g_f1"], golden["lane/g_f2"]
    idx, valid = golden["lane/g_idx"], golden["lane/g_valid"]
    got = O.pair_dots(f1, f2, np.arange(31), idx)
    want = golden["lane/gather"]
    assert np.array_equal(np.where(valid.astype(bool), got, np.float32(0)), want)
    at, bt = golden["lane/at"], golden["lane/bt"]
    mmm = np.stack([O.corr_pairs(at[q], bt[q]) for q in range(at.shape[0])])
    assert np.array_equal(mmm, golden["lane/mmm"])


def test_numpy_fallback_equals_c_helper(golden):
    a, b = golden["lane/a"], golden["lane/b"]
    ia = np.repeat(np.arange(23), 19)
    ib = np.tile(np.arange(19), 23)
    c = O.pair_dots(a, b, ia, ib)
    saved = O._CLIB
    O._CLIB = False
    try:
        n = O.pair_dots(a, b, ia, ib)
    finally:
        O._CLIB = saved
    assert np.array_equal(c, n)


@pytest.mark.parametrize("name", CASES)
def test_lookup_matches_golden(golden, name):
    r, L, norm = _spec(golden, name)
    f1, f2 = golden[f"{name}/f1"], golden[f"{name}/f2"]
    for it in range(int(golden[f"{name}/n_iter"])):
        got = O.lookup(f1, f2, golden[f"{name}/coords{it}"], r, L, norm)
        assert np.array_equal(got, golden[f"{name}/out{it}"]), (name, it)


@pytest.mark.parametrize("name", CASES)
def test_pool_volume_lookup_matches_golden(golden, name):
    r, L, norm = _spec(golden, name)
    f1, f2 = golden[f"{name}/f1"], golden[f"{name}/f2"]
    d = f1.shape[2]
    mats = [O.corr_pairs(f1.reshape(-1, d), f2.reshape(-1, d))]
    shapes = [f2.shape[:2]]
    for _ in range(1, L):
        mats.append(O.pool_volume(mats[-1], shapes[-1]))
        shapes.append((shapes[-1][0] // 2, shapes[-1][1] // 2))
    for lvl in range(L):
        ref = golden[f"{name}/pv_mat{lvl}"]
        if ref.size:
            assert np.array_equal(mats[lvl], ref)
    got = O.lookup_from_volume(mats, shapes, golden[f"{name}/coords0"], r, L, d, norm)
    assert np.array_equal(got, golden[f"{name}/dense_pv0"])


@pytest.mark.parametrize("name", CASES)
def test_ondemand_dot_count_matches_golden(golden, name):
    r, L, _ = _spec(golden, name)
    f2 = golden[f"{name}/f2"]
    coords = [golden[f"{name}/coords{it}"] for it in range(int(golden[f"{name}/n_iter"]))]
    assert O.ondemand_dot_count(coords, r, L, f2.shape[:2]) == int(golden[f"{name}/od_dots"])


def test_masks_and_block_ids_match_golden(golden):
    r, L, B, h, w = (int(v) for v in golden["mask/spec"])
    n_tgt = golden["mask/n_tgt"]
    cums = [np.zeros((int(golden["mask/n_src"]), int(n_tgt[l])), bool) for l in range(L)]
    used = [0] * L
    for it in range(3):
        c = golden[f"mask/coords{it}"]
        for lvl in range(L):
            m = O.mask_blocks(c, r, lvl, (h, w), B)
            assert np.array_equal(np.argwhere(m).astype(np.int32), golden[f"mask/m{it}_{lvl}"])
            pos, ids, cums[lvl] = O.block_indices(m, cums[lvl], used[lvl])
            assert np.array_equal(pos, golden[f"mask/pos{it}_{lvl}"])
            assert np.array_equal(ids, golden[f"mask/ids{it}_{lvl}"])
            used[lvl] += pos.size


def test_block_counters_match_golden(golden):
    """blocks_computed per iteration = sum of newly-set mask bits (sparse.py:343-345)."""
    name = "scen"
    r, L, _ = _spec(golden, name)
    h, w = golden[f"{name}/f1"].shape[:2]
    for B in (1, 4, 8):
        cum = None
        total = 0
        for it in range(int(golden[f"{name}/n_iter"])):
            c = golden[f"{name}/coords{it}"]
            masks = [O.mask_blocks(c, r, l, (h, w), B) for l in range(L)]
            if cum is None:
                cum = [np.zeros_like(m) for m in masks]
            for l in range(L):
                pos, _, cum[l] = O.block_indices(masks[l], cum[l], 0)
                total += pos.size
            assert total == int(golden[f"{name}/B{B}/blocks{it}"])


def test_oracle_matches_live_reference(reference):
    if reference is None:
        pytest.skip("oracle/_ref not built (reference source tree absent)")
    cv = reference
    rng = np.random.default_rng(123)
    for trial in range(6):
        h, w = int(rng.integers(3, 14)), int(rng.integers(3, 14))
        d, r, L = int(rng.integers(1, 20)), int(rng.integers(0, 4)), int(rng.integers(1, 3))
        if min(h, w) >> (L - 1) < 1:
            L = 1
        sc = cv.gen_scenario(trial, (h, w, d), 3, cv.LookupSpec(r, L, bool(trial % 2)))
        st = cv.init_state(sc.f1, sc.f2, sc.spec, int(rng.integers(1, 6)))
        for cf in sc.centroid_fields:
            want = cv.sample_iteration(st, cf).values
            got = O.lookup(sc.f1.values, sc.f2.values, cf.coords, r, L, sc.spec.normalize)
            assert np.array_equal(got, want)
