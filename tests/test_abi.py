"""The C-ABI library loads and exports every symbol include/corrvol_b200.h declares;
argument validation and status->exception mapping work without a GPU."""

import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "corrvol_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\*\s]+?)\b(cvb_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    for name in ("cvb_pool2x2", "cvb_build_pyramid", "cvb_corr_pairs", "cvb_corr_gather",
                 "cvb_block_mmm", "cvb_lookup_dense", "cvb_lookup_on_demand",
                 "cvb_partial_sample", "cvb_computation_mask", "cvb_block_indices"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2505_16942_b200 import _lib

    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    # and the Python binding covers the whole header
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_abi_version_and_launch_counter():
    from paper_2505_16942_b200 import _lib

    lib = _lib.load()
    assert lib.cvb_abi_version() == 2
    assert _lib.launch_count() >= 0


def test_invalid_arguments_raise_value_error_before_any_launch():
    from paper_2505_16942_b200 import _lib

    before = _lib.launch_count()
    with pytest.raises(ValueError, match="cannot 2x2-pool"):
        _lib.call("cvb_pool2x2", 1, 1, 4, 3, 1, None)
    with pytest.raises(ValueError):
        _lib.call("cvb_corr_pairs", 1, 4, 1, 4, 0, 1, 0, None)
    with pytest.raises(ValueError, match="empty level"):
        outs = (_lib._p * 3)(1, 1, 1)
        _lib.call("cvb_build_pyramid", 1, 3, 3, 2, 3, outs, None)
    assert _lib.launch_count() == before


def test_partial_sizes_host_only():
    from paper_2505_16942_b200 import _lib

    d = _lib.PartialDesc()
    d.h1, d.w1, d.d, d.levels, d.radius = 540, 960, 256, 4, 4
    for l, (c) in enumerate((24, 20, 16, 16)):
        d.cap_h[l] = d.cap_w[l] = c
        d.th[l], d.tw[l] = 540 >> l, 960 >> l
    nt, mi = C.c_int64(), C.c_int64()
    per = (C.c_int64 * 8)()
    _lib.call("cvb_partial_sizes", C.byref(d), C.byref(nt), C.byref(mi), per)
    assert nt.value == 68 * 120
    # per-level meta (8 ints per tile and level) + one 108-int plan record per tile
    assert mi.value == nt.value * 4 * 8 + (nt.value + 1) * 108
    assert per[0] == nt.value * 24 * 24 * 64
    f1b = C.c_int64()
    _lib.call("cvb_tc_sizes", C.byref(d), C.byref(f1b), per)
    assert f1b.value == nt.value * (64 * 256 * 4 + 64)  # B images + query exponents
    assert per[0] == 4 * 540 * 960 * 256 + 540 * 960  # hi/lo planes + cell exponents


def test_status_mapping():
    from paper_2505_16942_b200 import _lib
    from paper_2505_16942_b200.types import CacheLimitError, GatherMissError

    _lib.check(0)
    with pytest.raises(GatherMissError):
        _lib.check(2)
    with pytest.raises(CacheLimitError):
        _lib.check(3)
    with pytest.raises(RuntimeError):
        _lib.check(4)


def test_reference_facing_exports_exist():
    import paper_2505_16942_b200 as pkg

    for name in ("build_feature_pyramid", "build_volume_pyramid", "lookup_dense",
                 "lookup_on_demand", "init_state", "sample_iteration", "memory_footprint",
                 "set_computation_mask", "compute_block_indices", "sampled_block_mmm",
                 "gather_proxy", "count_work_on_demand", "estimate_dense_bytes", "pooled_dims",
                 "CorrSampler", "LookupSpec", "FeatureMap", "CentroidField", "CostMaps",
                 "WorkCounter", "GatherMissError", "CacheLimitError", "get_kernels"):
        assert hasattr(pkg, name), name
