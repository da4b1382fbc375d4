"""GPU parity: every CUDA entry point against the golden vectors (made by the
reference) and the CPU oracle.  STRICT arithmetic must be bit-identical;
fast arithmetic must hold both gates:
  reference gate  max|d| / (1 + max|ref|)           <= 1e-5 (harness.py:167-168)
  north-star gate max|d| / (max|F1_i| * max|F2_j|)  <= 1e-4 (BASELINE.json)
"""

import itertools

import numpy as np
import pytest
import torch

import paper_2505_16942_b200 as cvb
from oracle import corrvol_oracle as O

pytestmark = pytest.mark.gpu

CASES = ["small", "norm", "oob", "intr0", "padded", "scen", "d256", "nocache"]
REF_GATE = 1e-5
NS_GATE = 1e-4


def _spec(g, name):
    r, l, n = (int(v) for v in g[f"{name}/spec"])
    return cvb.LookupSpec(r, l, bool(n))


def _gates(got, want, f1, f2):
    return O.deviation(got, want, want), O.norm_gate(got, want, f1, f2)


def _case(g, name, dev):
    f1 = cvb.FeatureMap(torch.from_numpy(g[f"{name}/f1"]).to(dev))
    f2 = cvb.FeatureMap(torch.from_numpy(g[f"{name}/f2"]).to(dev))
    n = int(g[f"{name}/n_iter"])
    coords = [cvb.CentroidField(torch.from_numpy(g[f"{name}/coords{i}"]).to(dev)) for i in range(n)]
    outs = [g[f"{name}/out{i}"] for i in range(n)]
    return f1, f2, coords, outs


def test_pyramid_bit_exact(golden, cuda):
    for key in ("pyr", "pyr8"):
        f2 = cvb.FeatureMap(torch.from_numpy(golden[f"{key}/f2"]).to(cuda))
        pyr = cvb.build_feature_pyramid(f2, 3)
        for lvl in range(3):
            assert np.array_equal(pyr.levels[lvl].values.cpu().numpy(), golden[f"{key}/l{lvl}"])


def test_pyramid_bit_exact_large(cuda):
    rng = np.random.default_rng(0)
    f2 = rng.standard_normal((135, 241, 256)).astype(np.float32)
    pyr = cvb.build_feature_pyramid(cvb.FeatureMap(torch.from_numpy(f2).to(cuda)), 4)
    want = O.pyramid(f2, 4)
    for lvl in range(4):
        assert np.array_equal(pyr.levels[lvl].values.cpu().numpy(), want[lvl])


@pytest.mark.parametrize("shape", [(135, 241, 256), (37, 29, 20), (16, 16, 64)])
def test_fused_tc_prepare_pyramid_bit_exact(cuda, shape):
    """The tensor-core path builds pyramid levels >= 1 inside its operand
    split (cvb_tc_prepare + CVB_PREP_POOL): bit-exact with pool2x2."""
    rng = np.random.default_rng(1)
    h, w, d = shape
    f = lambda: cvb.FeatureMap(torch.from_numpy(
        rng.standard_normal((h, w, d)).astype(np.float32)).to(cuda))
    f1, f2 = f(), f()
    st = cvb.init_state(f1, f2, cvb.LookupSpec(4, 3))
    assert st.tc
    want = O.pyramid(f2.values.cpu().numpy(), 3)
    for lvl in range(3):
        assert np.array_equal(st.pyramid.levels[lvl].values.cpu().numpy(), want[lvl])
    # the fused pass (level-0 split inside the level-1 pooling, trailing
    # row / column separately) writes the same operand bytes as splitting
    # each level of a precomputed pyramid
    ref = cvb.init_state(f1, f2, cvb.LookupSpec(4, 3), pyramid=cvb.build_feature_pyramid(f2, 3))
    dp = -(-d // 64) * 64
    for lvl, (a, b) in enumerate(zip(st.tc_f2, ref.tc_f2)):
        cells = int(np.prod(st.pyramid.levels[lvl].values.shape[:2]))
        n = 4 * cells * dp + cells  # hi + lo planes + exponent bytes (the rest is padding)
        assert torch.equal(a[:n], b[:n])
    assert torch.equal(st.tc_f1, ref.tc_f1)


def test_floors_and_support_masks_bit_exact(golden, cuda):
    c = golden["floors/coords"]
    st_coords = cvb.CentroidField(torch.from_numpy(c).to(cuda))
    from paper_2505_16942_b200 import _lib
    from paper_2505_16942_b200._backend import stream_handle
    p = c.shape[0] * c.shape[1]
    for lvl in range(4):
        x0 = torch.empty(p, dtype=torch.int64, device=cuda)
        y0 = torch.empty_like(x0)
        fx = torch.empty(p, dtype=torch.float64, device=cuda)
        fy = torch.empty_like(fx)
        _lib.call("cvb_level_floors", _lib.ptr(st_coords.coords), p, lvl, _lib.CVB_COORDS_F64,
                  _lib.ptr(x0), _lib.ptr(y0), _lib.ptr(fx), _lib.ptr(fy), stream_handle())
        assert np.array_equal(x0.cpu().numpy(), golden[f"floors/x0_{lvl}"])
        assert np.array_equal(y0.cpu().numpy(), golden[f"floors/y0_{lvl}"])
        assert np.array_equal(fx.cpu().numpy(), golden[f"floors/fx_{lvl}"])
        assert np.array_equal(fy.cpu().numpy(), golden[f"floors/fy_{lvl}"])
        for gh, gw in ((7, 9), (16, 16)):
            r = 2
            out = torch.empty((p, (2 * r + 2) ** 2), dtype=torch.uint8, device=cuda)
            _lib.call("cvb_support_valid", _lib.ptr(st_coords.coords), p, lvl, r, gh, gw,
                      _lib.CVB_COORDS_F64, _lib.ptr(out), stream_handle())
            assert np.array_equal(out.cpu().numpy(), O.support_valid(c, lvl, r, gh, gw))


def test_kernel_lane_strict_bit_exact(golden, cuda):
    k = cvb.get_kernels("cuda")
    t = lambda a: torch.from_numpy(a).to(cuda)
    assert np.array_equal(k.corr_pairs(t(golden["lane/a"]), t(golden["lane/b"]), strict=True)
                          .cpu().numpy(), golden["lane/pairs"])
    g = k.corr_gather(t(golden["lane/g_f1"]), t(golden["lane/g_f2"]), t(golden["lane/g_idx"]),
                      t(golden["lane/g_valid"]), strict=True)
    assert np.array_equal(g.cpu().numpy(), golden["lane/gather"])
    m = k.block_mmm(t(golden["lane/at"]), t(golden["lane/bt"]), strict=True)
    assert np.array_equal(m.cpu().numpy(), golden["lane/mmm"])
    with pytest.raises(ValueError):
        cvb.get_kernels("cython")


def test_corr_pairs_large_strict_and_fast(cuda):
    rng = np.random.default_rng(1)
    a = rng.standard_normal((300, 256)).astype(np.float32)
    b = rng.standard_normal((190, 256)).astype(np.float32)
    want = O.corr_pairs(a, b)
    k = cvb.get_kernels()
    ta, tb = torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda)
    assert np.array_equal(k.corr_pairs(ta, tb, strict=True).cpu().numpy(), want)
    fast = k.corr_pairs(ta, tb).cpu().numpy()
    assert O.deviation(fast, want, want) <= REF_GATE


@pytest.mark.parametrize("name", CASES)
def test_ondemand_strict_bit_exact(golden, cuda, name):
    spec = _spec(golden, name)
    f1, f2, coords, outs = _case(golden, name, cuda)
    pyr = cvb.build_feature_pyramid(f2, spec.levels)
    counter = cvb.WorkCounter()
    for c, want in zip(coords, outs):
        got = cvb.lookup_on_demand(f1, pyr, c, spec, strict=True, counter=counter)
        assert np.array_equal(got.numpy(), want)
    assert counter.dot_products == int(golden[f"{name}/od_dots"])


@pytest.mark.parametrize("name", CASES)
def test_dense_strict_bit_exact(golden, cuda, name):
    spec = _spec(golden, name)
    f1, f2, coords, outs = _case(golden, name, cuda)
    vol = cvb.build_volume_pyramid(f1, f2, spec.levels, mode="pool_features", strict=True)
    for c, want in zip(coords, outs):
        assert np.array_equal(cvb.lookup_dense(vol, c, spec, strict=True).numpy(), want)
    vol_pv = cvb.build_volume_pyramid(f1, f2, spec.levels, mode="pool_volume", strict=True)
    for lvl in range(spec.levels):
        ref = golden[f"{name}/pv_mat{lvl}"]
        if ref.size:
            assert np.array_equal(vol_pv.level_mats[lvl].cpu().numpy(), ref)
    got = cvb.lookup_dense(vol_pv, coords[0], spec, strict=True).numpy()
    assert np.array_equal(got, golden[f"{name}/dense_pv0"])


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("mode", ["pool_features", "pool_volume"])
def test_dense_tc_volume_within_gates(golden, cuda, name, mode):
    """Fast dense volume (tcgen05 split-fp16, cvb_dense_tc): every level matrix
    within the north-star gate of the strict (reference-exact) volume, and
    lookups within both gates of the reference outputs."""
    spec = _spec(golden, name)
    f1, f2, coords, outs = _case(golden, name, cuda)
    fast = cvb.build_volume_pyramid(f1, f2, spec.levels, mode=mode)
    strict = cvb.build_volume_pyramid(f1, f2, spec.levels, mode=mode, strict=True)
    n1 = float(torch.linalg.vector_norm(f1.values, dim=-1).max())
    n2 = float(torch.linalg.vector_norm(f2.values, dim=-1).max())
    for a, b in zip(fast.level_mats, strict.level_mats):
        assert a.shape == b.shape
        if a.numel():
            assert float((a - b).abs().max()) <= NS_GATE * n1 * n2
    if mode == "pool_features":
        for c, want in zip(coords, outs):
            got = cvb.lookup_dense(fast, c, spec).numpy()
            ref_dev, ns_dev = _gates(got, want, golden[f"{name}/f1"], golden[f"{name}/f2"])
            assert ref_dev <= REF_GATE and ns_dev <= NS_GATE, (ref_dev, ns_dev)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("mode", ["tile", "block"])
def test_partial_strict_bit_exact(golden, cuda, name, mode):
    spec = _spec(golden, name)
    f1, f2, coords, outs = _case(golden, name, cuda)
    blocks = [int(k.split("/")[1][1:]) for k in golden if k.startswith(f"{name}/B")
              and k.endswith("/footprint")]
    cache = name != "nocache"
    for B in (blocks or [2]):
        st = cvb.init_state(f1, f2, spec, B, mode=mode, strict=True, cache_enabled=cache)
        for it, (c, want) in enumerate(zip(coords, outs)):
            got = cvb.sample_iteration(st, c)
            assert np.array_equal(got.numpy(), want), (name, mode, B, it)
            if mode == "block" and blocks:
                assert st.counter.blocks_computed == int(golden[f"{name}/B{B}/blocks{it}"])
                assert [lv.store.used for lv in st.levels] == \
                    list(golden[f"{name}/B{B}/used{it}"])
                assert [int(lv.mask_union.sum()) for lv in st.levels] == \
                    list(golden[f"{name}/B{B}/union{it}"])
        if mode == "block" and blocks:
            for lvl, lv in enumerate(st.levels):
                ids = lv.block_ids.cpu().numpy().ravel()
                nz = np.flatnonzero(ids >= 0)
                assert np.array_equal(np.stack([nz, ids[nz]]).astype(np.int32),
                                      golden[f"{name}/B{B}/ids_l{lvl}"])
            fp = cvb.memory_footprint(st)
            want_fp = golden[f"{name}/B{B}/footprint"]
            assert [fp["mask_bytes"], fp["block_bytes"], fp["capacity_bytes"],
                    fp["blocks_used"]] == list(want_fp)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("variant", ["partial", "ondemand", "dense"])
def test_fast_variants_within_tolerance(golden, cuda, name, variant):
    spec = _spec(golden, name)
    f1, f2, coords, outs = _case(golden, name, cuda)
    s = cvb.CorrSampler(f1, f2, spec, variant=variant)
    for c, want in zip(coords, outs):
        got = s(c).numpy()
        ref_dev, ns_dev = _gates(got, want, golden[f"{name}/f1"], golden[f"{name}/f2"])
        assert ref_dev <= REF_GATE and ns_dev <= NS_GATE, (ref_dev, ns_dev)


def test_masks_and_block_ids_bit_exact(golden, cuda):
    r, L, B, h, w = (int(v) for v in golden["mask/spec"])
    rng = np.random.default_rng(0)
    f = lambda s: cvb.FeatureMap(torch.from_numpy(
        rng.standard_normal(s).astype(np.float32)).to(cuda))
    st = cvb.init_state(f((h, w, 4)), f((h, w, 4)), cvb.LookupSpec(r, L), B, mode="block",
                        strict=True)
    for it in range(3):
        c = cvb.CentroidField(torch.from_numpy(golden[f"mask/coords{it}"]).to(cuda))
        for lvl in range(L):
            m = cvb.set_computation_mask(st, c, lvl)
            assert np.array_equal(np.argwhere(m.cpu().numpy()).astype(np.int32),
                                  golden[f"mask/m{it}_{lvl}"])
            pos, ids = cvb.compute_block_indices(st, m, lvl)
            assert np.array_equal(pos.cpu().numpy(), golden[f"mask/pos{it}_{lvl}"])
            assert np.array_equal(ids.cpu().numpy(), golden[f"mask/ids{it}_{lvl}"])
            cvb.sampled_block_mmm(st, lvl, pos)


def test_block_mode_errors(cuda):
    rng = np.random.default_rng(3)
    f = lambda s: cvb.FeatureMap(torch.from_numpy(
        rng.standard_normal(s).astype(np.float32)).to(cuda))
    st = cvb.init_state(f((8, 8, 2)), f((8, 8, 2)), cvb.LookupSpec(2, 1), 2, mode="block",
                        hard_limit_bytes=2 * 4 * 16)
    ys, xs = np.mgrid[0:8, 0:8]
    c = cvb.CentroidField(np.stack([xs, ys], -1).astype(np.float64) + 0.3)
    with pytest.raises(cvb.CacheLimitError):
        cvb.sample_iteration(st, c)
    # transactional: state untouched by the failed iteration
    assert all(lv.store.used == 0 for lv in st.levels)
    assert all(int(lv.mask_cum.sum()) == 0 for lv in st.levels)
    with pytest.raises(cvb.GatherMissError):
        cvb.gather_proxy(st, 0, 0, (1.5, 1.5))


def _acceptance_params():
    """The reference's 104 acceptance scenarios (test_acceptance.py:71-108)."""
    rng = np.random.default_rng(20260816)
    blocks = itertools.cycle((1, 2, 4, 8))
    params = []

    def add(h, w, d, r, l, n):
        params.append(dict(seed=1000 + len(params), dims=(int(h), int(w), int(d)),
                           radius=int(r), levels=int(l), iterations=int(n), block=next(blocks)))

    for _ in range(64):
        add(rng.integers(4, 13), rng.integers(4, 13), rng.integers(3, 17), rng.integers(1, 3),
            rng.integers(1, 3), rng.integers(1, 7))
    for _ in range(30):
        add(rng.integers(13, 25), rng.integers(13, 25), rng.integers(8, 33), rng.integers(2, 5),
            rng.integers(2, 4), rng.integers(4, 11))
    for _ in range(8):
        add(rng.integers(25, 33), rng.integers(25, 33), rng.integers(16, 65), 4, 4,
            rng.integers(8, 17))
    add(4, 32, 8, 2, 2, 6)
    add(32, 4, 8, 2, 2, 6)
    return params


def test_acceptance_suite_three_way(cuda):
    """Criterion 01 on the GPU: all variants bitwise (strict) / within 1e-5 (fast)."""
    params = _acceptance_params()
    assert len(params) >= 100
    worst = 0.0
    for p in params:
        spec = cvb.LookupSpec(p["radius"], p["levels"])
        sc = cvb.gen_scenario(p["seed"], p["dims"], p["iterations"], spec)
        f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(cuda))
        f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(cuda))
        strict_tile = cvb.init_state(f1, f2, spec, p["block"], strict=True)
        strict_block = cvb.init_state(f1, f2, spec, p["block"], mode="block", strict=True)
        fast = cvb.CorrSampler(f1, f2, spec, variant="partial")
        pyr = strict_tile.pyramid
        for coords in sc.centroid_fields:
            want = O.lookup(sc.f1, sc.f2, coords, spec.radius, spec.levels)
            c = cvb.CentroidField(torch.from_numpy(coords).to(cuda))
            assert np.array_equal(cvb.sample_iteration(strict_tile, c).numpy(), want), p
            assert np.array_equal(cvb.sample_iteration(strict_block, c).numpy(), want), p
            assert np.array_equal(
                cvb.lookup_on_demand(f1, pyr, c, spec, strict=True).numpy(), want), p
            got = fast(c).numpy()
            worst = max(worst, O.deviation(got, want, want))
    assert worst <= REF_GATE


def test_tile_overflow_and_no_cache_paths_bitwise(cuda):
    """Tiny cache windows force the direct path; cache-off recomputes — same bits."""
    spec = cvb.LookupSpec(4, 3)
    sc = cvb.gen_scenario(3, (40, 52, 32), 5, spec)
    f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(cuda))
    f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(cuda))
    a = cvb.init_state(f1, f2, spec, strict=True)
    b = cvb.init_state(f1, f2, spec, strict=True, tile_caps=(18, 14, 12))
    c = cvb.init_state(f1, f2, spec, strict=True, cache_enabled=False)
    for coords in sc.centroid_fields:
        want = O.lookup(sc.f1, sc.f2, coords, 4, 3)
        cc = cvb.CentroidField(torch.from_numpy(coords).to(cuda))
        for st in (a, b, c):
            assert np.array_equal(cvb.sample_iteration(st, cc).numpy(), want)
    assert b.device_counters["overflow_tile_levels"] > 0
    assert c.device_counters["cells"] > a.device_counters["cells"]


def test_float32_coords_match_float64_reference(cuda):
    spec = cvb.LookupSpec(4, 2, True)
    sc = cvb.gen_scenario(9, (24, 31, 16), 3, spec, coords_dtype=np.float32)
    f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(cuda))
    f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(cuda))
    st = cvb.init_state(f1, f2, spec, strict=True)
    for coords in sc.centroid_fields:
        c32 = cvb.CentroidField(torch.from_numpy(coords).to(cuda))
        assert c32.coords.dtype == torch.float32
        want = O.lookup(sc.f1, sc.f2, coords.astype(np.float64), 4, 2, True)
        assert np.array_equal(cvb.sample_iteration(st, c32).numpy(), want)


@pytest.mark.parametrize("spread", [6.0, 14.0])
def test_divergent_flow_group_split_and_overflow(cuda, spread):
    """Random per-pixel displacements: query rows whose supports do not fit one
    staged region (group split / per-query fallback) and tile boxes larger than
    the cache window (overflow path) must still be bit-exact (strict) and
    within tolerance (fast)."""
    rng = np.random.default_rng(int(spread))
    h, w, d = 33, 47, 24
    spec = cvb.LookupSpec(4, 3)
    f1n = rng.standard_normal((h, w, d)).astype(np.float32)
    f2n = rng.standard_normal((h, w, d)).astype(np.float32)
    f1 = cvb.FeatureMap(torch.from_numpy(f1n).to(cuda))
    f2 = cvb.FeatureMap(torch.from_numpy(f2n).to(cuda))
    strict = cvb.init_state(f1, f2, spec, strict=True)
    fast = cvb.init_state(f1, f2, spec)
    ys, xs = np.mgrid[0:h, 0:w]
    base = np.stack([xs, ys], -1).astype(np.float64)
    for it in range(3):
        coords = base + rng.uniform(-spread, spread, size=base.shape)
        want = O.lookup(f1n, f2n, coords, 4, 3)
        c = cvb.CentroidField(torch.from_numpy(coords).to(cuda))
        assert np.array_equal(cvb.sample_iteration(strict, c).numpy(), want)
        got = cvb.sample_iteration(fast, c).numpy()
        assert O.deviation(got, want, want) <= REF_GATE
    if spread > 10:
        assert strict.device_counters["overflow_tile_levels"] > 0


def test_pipelined_tile_ranges_equal_single_launch(cuda):
    """Contract/gather over tile ranges on two streams == one launch, bit for bit."""
    spec = cvb.LookupSpec(4, 4)
    sc = cvb.gen_scenario(4, (70, 90, 64), 4, spec, coords_dtype=np.float32)
    f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(cuda))
    f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(cuda))
    one = cvb.init_state(f1, f2, spec, pipeline_splits=1)
    many = cvb.init_state(f1, f2, spec, pipeline_splits=5)
    assert one.tc and many.pipeline_splits == 5
    for coords in sc.centroid_fields:
        c = cvb.CentroidField(torch.from_numpy(coords).to(cuda))
        a = cvb.sample_iteration(one, c).numpy()
        b = cvb.sample_iteration(many, c).numpy()
        assert np.array_equal(a, b)
        want = O.lookup(sc.f1, sc.f2, coords, 4, 4)
        assert O.deviation(b, want, want) <= REF_GATE


@pytest.mark.parametrize("levels,radius", [(5, 4), (6, 3)])
def test_more_levels_than_one_sampler_launch(cuda, levels, radius):
    """Pyramids deeper than the SM-pair kernel and one fast-sampler launch take
    (4 levels): the cold iteration on the single-tile kernel, the r=4 sampler
    in two launches (levels 0-3, then the rest), the generic-radius sampler
    for r=3.  Strict bit for bit, fast within both gates, every iteration."""
    spec = cvb.LookupSpec(radius, levels)
    sc = cvb.gen_scenario(11, (96, 160, 64), 4, spec, coords_dtype=np.float32)
    f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(cuda))
    f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(cuda))
    strict = cvb.CorrSampler(f1, f2, spec, strict=True)
    fast = cvb.CorrSampler(f1, f2, spec)
    assert fast.state.tc
    for coords in sc.centroid_fields:
        want = O.lookup(sc.f1, sc.f2, coords, radius, levels)
        c = cvb.CentroidField(torch.from_numpy(coords).to(cuda))
        assert np.array_equal(strict(c).numpy(), want)
        dev, ns = _gates(fast(c).numpy(), want, sc.f1, sc.f2)
        assert dev <= REF_GATE and ns <= NS_GATE


@pytest.mark.parametrize("split", ["row_aligned", "mid_row"])
def test_disjoint_ranges_contract_concurrently(cuda, split):
    """include/corrvol_b200.h: disjoint tile ranges may run concurrently.  Two
    ranges contracted and gathered on two streams at once, every iteration
    (a mid-row split also puts the cold iteration on the single-tile kernel
    instead of the SM pairs) == one launch over the frame, bit for bit."""
    from paper_2505_16942_b200 import _lib, sparse
    from paper_2505_16942_b200.dense import coords_flags
    spec = cvb.LookupSpec(4, 4)
    sc = cvb.gen_scenario(6, (72, 104, 64), 5, spec, coords_dtype=np.float32)
    f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(cuda))
    f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(cuda))
    ref = cvb.init_state(f1, f2, spec)
    st = cvb.init_state(f1, f2, spec)
    n, tx = st.n_tiles, -(-104 // 8)
    k = (n // tx // 2) * tx if split == "row_aligned" else n // 2 + 3
    full = st.desc
    ranges = []
    for a, b in ((0, k), (k, n)):
        d = _lib.PartialDesc()
        _lib.C.pointer(d)[0] = full
        d.tile_begin, d.tile_end = a, b
        ranges.append(d)
    streams = [torch.cuda.Stream(cuda), torch.cuda.Stream(cuda)]
    main = torch.cuda.current_stream(cuda)
    for coords in sc.centroid_fields:
        c = cvb.CentroidField(torch.from_numpy(coords).to(cuda))
        want = cvb.sample_iteration(ref, c).numpy()
        out = torch.empty((72, 104, 4, 9, 9), dtype=torch.float32, device=cuda)
        flags = coords_flags(c, False)
        f2s, caches = sparse._contract_args(st, c, flags)
        ev = torch.cuda.Event()
        ev.record(main)
        try:
            for d, s in zip(ranges, streams):
                s.wait_event(ev)
                with torch.cuda.stream(s):
                    st.desc = d
                    sparse._contract(st, c, flags, f2s, caches)
                    sparse._gather(st, c, flags, f2s, caches, out)
        finally:
            st.desc = full
        for s in streams:
            main.wait_stream(s)
        st.iteration += 1
        assert np.array_equal(out.cpu().numpy(), want)


def test_tc_per_row_scaling_wide_dynamic_range(cuda):
    """Rows spanning 2^-20 .. 2^20 in magnitude: every row carries its own
    power-of-two scale through the fp16 split, so both gates hold per row."""
    rng = np.random.default_rng(5)
    h, w, d = 24, 40, 256
    scale1 = np.exp2(rng.integers(-20, 21, size=(h, w, 1))).astype(np.float32)
    scale2 = np.exp2(rng.integers(-20, 21, size=(h, w, 1))).astype(np.float32)
    f1 = (rng.standard_normal((h, w, d)) * scale1).astype(np.float32)
    f2 = (rng.standard_normal((h, w, d)) * scale2).astype(np.float32)
    spec = cvb.LookupSpec(4, 2)
    sc = cvb.gen_scenario(3, (h, w, 4), 2, spec, coords_dtype=np.float32)
    s = cvb.CorrSampler(cvb.FeatureMap(torch.from_numpy(f1).to(cuda)),
                        cvb.FeatureMap(torch.from_numpy(f2).to(cuda)), spec)
    for c in sc.centroid_fields:
        want = O.lookup(f1, f2, c, spec.radius, spec.levels)
        got = s(cvb.CentroidField(torch.from_numpy(c).to(cuda))).numpy()
        # per-query relative error against the query's own cost scale
        err = np.abs(got - want).reshape(h * w, -1).max(axis=1)
        ref = np.abs(want).reshape(h * w, -1).max(axis=1)
        ok = ref > 0
        assert np.all(err[ok] <= 1e-5 * (ref[ok] + np.finfo(np.float32).tiny) * 16)


@pytest.mark.parametrize("strict", [False, True])
def test_row_bands_concatenate_to_full_frame_bitwise(cuda, strict):
    """query-row bands (starts aligned to the 8-row tile) against a
    replicated fmap2 reproduce the single-GPU frame bit for bit."""
    from paper_2505_16942_b200.parallel import row_bands

    spec = cvb.LookupSpec(4, 4)
    h, w, d = 70, 90, 64
    sc = cvb.gen_scenario(6, (h, w, d), 3, spec, coords_dtype=np.float32)
    f1 = torch.from_numpy(sc.f1).to(cuda)
    f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(cuda))
    full = cvb.CorrSampler(cvb.FeatureMap(f1), f2, spec, strict=strict)
    bands = [cvb.CorrSampler(cvb.FeatureMap(f1[a:b].contiguous()), f2, spec, strict=strict)
             for a, b in row_bands(h, 3)]
    for c in sc.centroid_fields:
        ct = torch.from_numpy(c).to(cuda)
        want = full(cvb.CentroidField(ct)).numpy()
        got = np.concatenate([s(cvb.CentroidField(ct[a:b].contiguous())).numpy()
                              for s, (a, b) in zip(bands, row_bands(h, 3))])
        assert np.array_equal(got, want)


def test_batch_sampler_equals_per_pair(cuda):
    spec = cvb.LookupSpec(4, 3)
    scs = [cvb.gen_scenario(s, (24, 40, 32), 2, spec, coords_dtype=np.float32) for s in (1, 2, 3)]
    f1 = torch.stack([torch.from_numpy(s.f1) for s in scs]).to(cuda)
    f2 = torch.stack([torch.from_numpy(s.f2) for s in scs]).to(cuda)
    batch = cvb.BatchCorrSampler(f1, f2, spec)
    singles = [cvb.CorrSampler(cvb.FeatureMap(f1[i]), cvb.FeatureMap(f2[i]), spec)
               for i in range(3)]
    for it in range(2):
        coords = torch.stack([torch.from_numpy(s.centroid_fields[it]) for s in scs]).to(cuda)
        got = batch(coords).cpu().numpy()
        for i in range(3):
            assert np.array_equal(got[i], singles[i](cvb.CentroidField(coords[i])).numpy())


def test_graph_mode_equals_eager(cuda):
    """CorrSampler(graph=True) replays captured iterations: same results."""
    spec = cvb.LookupSpec(4, 4)
    sc = cvb.gen_scenario(8, (46, 62, 64), 5, spec, coords_dtype=np.float32)
    f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(cuda))
    f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(cuda))
    eager = cvb.CorrSampler(f1, f2, spec)
    graphed = cvb.CorrSampler(f1, f2, spec, graph=True)
    for c in sc.centroid_fields:
        ct = torch.from_numpy(c).to(cuda)
        want = eager(cvb.CentroidField(ct)).values.clone()
        got = graphed(cvb.CentroidField(ct)).values
        assert torch.equal(got, want)
    assert graphed._graph is not None and graphed.state.iteration == 5


@pytest.mark.parametrize("d,tc", [(256, True), (264, False), (320, False)])
def test_feature_width_selects_contraction_and_holds_gates(cuda, d, tc):
    """D <= 256 contracts on tcgen05 (split fp16); wider features take the FP32
    FFMA contraction of the same tiler — both within the reference gates."""
    spec = cvb.LookupSpec(4, 3)
    sc = cvb.gen_scenario(5, (24, 40, d), 3, spec)
    f1 = cvb.FeatureMap(torch.from_numpy(sc.f1).to(cuda))
    f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(cuda))
    st = cvb.init_state(f1, f2, spec)
    assert st.tc == tc
    for coords in sc.centroid_fields:
        want = O.lookup(sc.f1, sc.f2, coords, spec.radius, spec.levels)
        got = cvb.sample_iteration(st, cvb.CentroidField(torch.from_numpy(coords).to(cuda))).numpy()
        dev_, ns = _gates(got, want, sc.f1, sc.f2)
        assert dev_ <= REF_GATE and ns <= NS_GATE, (d, dev_, ns)
