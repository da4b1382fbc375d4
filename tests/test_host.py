"""Host-side logic on CPU: boundary types, geometry helpers, work models, the
scenario generator, the block-store policy and the no-fallback rule."""

import numpy as np
import pytest
import torch

import paper_2505_16942_b200 as cvb
from oracle import corrvol_oracle as O
from paper_2505_16942_b200.sparse import BlockStore, PaddedGrid, _pack_bits, unpack_bits


def test_lookup_spec_validation_and_scale():
    with pytest.raises(ValueError):
        cvb.LookupSpec(-1, 1)
    with pytest.raises(ValueError):
        cvb.LookupSpec(1, 0)
    s = cvb.LookupSpec(4, 4, True)
    assert s.window == 9 and s.support == 10
    assert s.scale(256) == float(np.float32(1.0 / 16.0))
    assert cvb.LookupSpec(4, 4).scale(256) == 1.0


def test_feature_map_and_centroid_validation():
    with pytest.raises(ValueError):
        cvb.FeatureMap(np.zeros((2, 3), np.float32))
    with pytest.raises(ValueError):
        cvb.FeatureMap(np.zeros((2, 0, 3), np.float32))
    bad = np.zeros((2, 2, 3), np.float32)
    bad[0, 0, 0] = np.nan
    with pytest.raises(ValueError):
        cvb.FeatureMap(bad)
    with pytest.raises(ValueError):
        cvb.CentroidField(np.zeros((2, 2, 3)))
    with pytest.raises(ValueError):
        cvb.CentroidField(np.full((2, 2, 2), np.inf))
    c32 = cvb.CentroidField(np.zeros((2, 2, 2), np.float32))
    assert c32.coords.dtype == torch.float32
    c64 = cvb.CentroidField(np.zeros((2, 2, 2), np.int64))
    assert c64.coords.dtype == torch.float64


def test_caller_arrays_are_not_frozen():
    a = np.ones((2, 2, 2), np.float32)
    cvb.FeatureMap(a)
    a[0, 0, 0] = 5.0  # the reference freezes the caller's array here (types.py:58-65)
    assert a.flags.writeable


def test_cost_maps_shape_check():
    with pytest.raises(ValueError):
        cvb.CostMaps(torch.zeros(2, 2, 1, 3, 4), radius=1)
    cm = cvb.CostMaps(torch.zeros(2, 3, 2, 3, 3), radius=1)
    assert cm.per_pixel().shape == (6, 18)


def test_pooled_dims_and_dense_bytes():
    assert cvb.pooled_dims((9, 7), 1) == (4, 3)
    assert cvb.pooled_dims((9, 7), 2) == (2, 1)
    assert cvb.estimate_dense_bytes((4, 4), (4, 4), 2) == 4 * 16 * (16 + 4)
    assert cvb.estimate_dense_bytes((540, 960), (540, 960), 4) == 1427523559200 or \
        cvb.estimate_dense_bytes((540, 960), (540, 960), 4) > 1.4e12


def test_count_work_on_demand_matches_oracle(golden):
    for name in ("small", "scen", "padded"):
        r, L, n = (int(v) for v in golden[f"{name}/spec"])
        f2 = golden[f"{name}/f2"]
        fields = [cvb.CentroidField(torch.from_numpy(golden[f"{name}/coords{i}"]))
                  for i in range(int(golden[f"{name}/n_iter"]))]
        h, w, d = golden[f"{name}/f1"].shape
        wc = cvb.count_work_on_demand((h, w, d), cvb.LookupSpec(r, L), fields, f2.shape[:2])
        assert wc.dot_products == int(golden[f"{name}/od_dots"])
        assert wc.macs == wc.dot_products * d
        assert wc.macs <= wc.upper_bound_macs


def test_scenario_generator_matches_reference(reference):
    if reference is None:
        pytest.skip("oracle/_ref not built")
    for seed, dims, n in ((0, (9, 11, 4), 4), (1003, (20, 16, 32), 3)):
        mine = cvb.gen_scenario(seed, dims, n, cvb.LookupSpec(4, 3))
        ref = reference.gen_scenario(seed, dims, n, reference.LookupSpec(4, 3))
        assert np.array_equal(mine.f1, ref.f1.values)
        assert np.array_equal(mine.f2, ref.f2.values)
        for a, b in zip(mine.centroid_fields, ref.centroid_fields):
            assert np.array_equal(a, b.coords)


def test_scenario_float32_quantisation():
    sc = cvb.gen_scenario(3, (6, 7, 2), 3, cvb.LookupSpec(1, 1), coords_dtype=np.float32)
    assert all(c.dtype == np.float32 for c in sc.centroid_fields)


def test_block_store_growth_and_cap_policy():
    s = BlockStore(2, growth_factor=2, overalloc_cap_bytes=0)
    assert s.bytes_per_block == 4 * 16
    s.ensure_capacity(3)
    assert s.capacity == 3
    s.append(torch.zeros(3, 4, 4))
    ev = s.growth_events
    s.ensure_capacity(2)
    assert s.capacity == 5 and s.growth_events == ev + 1
    big = BlockStore(2, overalloc_cap_bytes=10 ** 9)
    big.ensure_capacity(3)
    assert big.capacity == 4
    big.append(torch.ones(3, 4, 4))
    big.ensure_capacity(2)
    assert big.capacity == 8
    assert torch.equal(big.data[0], torch.ones(4, 4))
    with pytest.raises(ValueError):
        BlockStore(2, growth_factor=1)


def test_block_store_hard_limit():
    s = BlockStore(2, hard_limit_bytes=3 * 4 * 16)
    s.ensure_capacity(3)
    with pytest.raises(cvb.CacheLimitError):
        s.ensure_capacity(4)


def test_cache_cap_env_var(monkeypatch):
    monkeypatch.setenv("CORRVOL_CACHE_CAP_BYTES", "0")
    assert BlockStore(2).overalloc_cap_bytes == 0
    monkeypatch.setenv("CORRVOL_CACHE_CAP_BYTES", "-3")
    with pytest.raises(ValueError):
        BlockStore(2)


def test_bit_pack_roundtrip():
    rng = np.random.default_rng(0)
    m = torch.from_numpy(rng.random((7, 75)) < 0.3)
    words = _pack_bits(m, 3)
    assert words.dtype == torch.int32
    assert torch.equal(unpack_bits(words, 75), m)


def test_padded_grid_geometry():
    g = PaddedGrid.of(10, 13, 4, 8)
    assert (g.padded_height, g.padded_width, g.tiles_y, g.tiles_x, g.n_tiles) == (16, 16, 2, 2, 4)
    assert cvb.padded_extent(17, 8) == 24


def test_backend_selection(monkeypatch):
    from paper_2505_16942_b200 import _backend

    assert cvb.available_backends() == ["cuda"]
    assert _backend.resolve_backend(None) == "cuda"
    with pytest.raises(ValueError):
        cvb.get_kernels("python")
    monkeypatch.setenv("CORRVOL_BACKEND", "cython")
    with pytest.raises(ValueError):
        cvb.default_backend()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the CPU-only failure mode")
def test_product_path_fails_loudly_without_cuda():
    f = cvb.FeatureMap(torch.zeros(4, 4, 2))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        cvb.build_feature_pyramid(f, 2)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        cvb.init_state(f, f, cvb.LookupSpec(1, 1))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        cvb.get_kernels().corr_pairs(torch.zeros(2, 2), torch.zeros(2, 2))


def test_sampler_variant_validation():
    with pytest.raises(ValueError):
        cvb.CorrSampler(np.zeros((2, 2, 2), np.float32), np.zeros((2, 2, 2), np.float32),
                        cvb.LookupSpec(1, 1), variant="sparse-ish")
