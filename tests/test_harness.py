"""GPU harness: the reference's counter-based
acceptance criteria re-asserted on GPU counters, and the reference's CSV
schemas reproduced byte for byte."""

import csv
import io

import numpy as np
import pytest

import paper_2505_16942_b200 as cvb
from paper_2505_16942_b200 import harness as H
from oracle import import_reference


def _rec(**kw):
    base = dict(sampler="sparse", backend="cuda", height=16, width=24, feature_dim=8, radius=4,
                levels=2, block=4, iterations=3, cache="on", seed=5, dot_products=123,
                macs=984, blocks_computed=7, blocks_stored=7, blocks_union=9,
                block_positions=60, peak_bytes=4096, wall_ms=1.25, shares=None, oom=False)
    base.update(kw)
    return base


def test_bench_csv_matches_reference_format():
    ref = import_reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from corrvol.harness import BenchRecord as RefRecord, bench_csv as ref_csv

    rows = [_rec(), _rec(sampler="dense", cache="", oom=True, wall_ms=0.0),
            _rec(shares={"mask": 10.0, "indices": 5.0, "mmm": 50.0, "cache": 5.0,
                         "sampling": 30.0})]
    ours = H.bench_csv([H.BenchRecord(**r) for r in rows])
    theirs = ref_csv([RefRecord(**r) for r in rows])
    assert ours == theirs


def test_equivalence_csv_matches_reference_format():
    ref = import_reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from corrvol.harness import EquivalenceReport as RefReport, equivalence_csv as ref_csv

    rows = [{"iteration": 0, "dev_dense_ondemand": 1.5e-7, "dev_dense_sparse": 0.0,
             "dev_ondemand_sparse": 2e-8, "bitwise_ondemand": True, "bitwise_sparse": False,
             "new_blocks": 12}]
    ours = H.equivalence_csv(H.EquivalenceReport(4, 1e-5, 1, rows, 1.5e-7, True, False, True))
    theirs = ref_csv(RefReport(4, 1e-5, 1, rows, 1.5e-7, True, False, True, None))
    assert ours == theirs


@pytest.mark.gpu
def test_gpu_equivalence_three_way(cuda):
    """Criterion 01 shape: ondemand and sparse bitwise equal to the
    feature-pooled dense build (strict), all within 1e-5 of the volume-pooled
    build."""
    for seed, (h, w, d), b in [(1, (24, 20, 16), 4), (2, (17, 33, 8), 8), (3, (16, 16, 32), 1)]:
        sc = cvb.gen_scenario(seed, (h, w, d), 4, cvb.LookupSpec(4, 3))
        rep = H.run_equivalence(sc, b)
        assert rep.passed and rep.bitwise_ondemand and rep.bitwise_sparse, rep.per_iteration


@pytest.mark.gpu
def test_gpu_equivalence_matches_reference_counters(cuda):
    """new_blocks per iteration equal the reference's run_equivalence."""
    ref = import_reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from corrvol.harness import gen_scenario as ref_gen, run_equivalence as ref_eq

    ours_sc = cvb.gen_scenario(3, (32, 32, 8), 6, cvb.LookupSpec(4, 2))
    theirs = ref_eq(ref_gen(3, (32, 32, 8), 6, ref.LookupSpec(4, 2)), 4)
    ours = H.run_equivalence(ours_sc, 4)
    assert [r["new_blocks"] for r in ours.per_iteration] == \
        [r["new_blocks"] for r in theirs.per_iteration]


@pytest.mark.gpu
def test_criterion_05_memory_scaling_exponent(cuda):
    spec = cvb.LookupSpec(4, 4)
    peaks = []
    sides = (32, 64, 128, 256)
    for side in sides:
        block = int(round((side * side) ** 0.125))
        sc = cvb.gen_scenario(100 + side, (side, side, 8), 8, spec)
        (rec,) = H.run_bench(sc, samplers=("sparse",), block_sizes=(block,))
        assert not rec.oom
        peaks.append(rec.peak_bytes)
    slope = float(np.polyfit(np.log([s * s for s in sides]), np.log(peaks), 1)[0])
    assert slope <= 1.7 and slope < 2.0


@pytest.mark.gpu
def test_criterion_06_caching_effectiveness(cuda):
    spec = cvb.LookupSpec(4, 2)
    sc = cvb.gen_scenario(3, (32, 32, 8), 16, spec)
    recs = H.run_bench(sc, samplers=("sparse", "partial"), block_sizes=(4,),
                       cache_modes=(True, False))
    for sampler, counter in (("sparse", "blocks_computed"), ("partial", "dot_products")):
        on = next(r for r in recs if r.sampler == sampler and r.cache == "on")
        off = next(r for r in recs if r.sampler == sampler and r.cache == "off")
        assert getattr(on, counter) <= 0.70 * getattr(off, counter)
    rep = H.run_equivalence(sc, 4)
    assert rep.per_iteration[1]["new_blocks"] < rep.per_iteration[0]["new_blocks"]


@pytest.mark.gpu
def test_criterion_07_work_savings_bound(cuda):
    spec = cvb.LookupSpec(4, 2)
    checked = 0
    for side in (16, 32, 64):
        sc = cvb.gen_scenario(side, (side, side, 8), 16, spec)
        recs = H.run_bench(sc, samplers=("dense", "sparse"), block_sizes=(1, 2, 4, 8))
        dense = next(r for r in recs if r.sampler == "dense")
        assert not dense.oom
        for r in recs:
            if r.sampler != "sparse":
                continue
            bound = r.blocks_union / r.block_positions * dense.dot_products * (1 + 1 / r.block)
            assert r.dot_products <= bound
            checked += 1
    assert checked == 12


@pytest.mark.gpu
def test_criterion_10_dense_quadratic_growth_from_csv(cuda):
    recs = []
    for side in (16, 32, 64):
        sc = cvb.gen_scenario(side, (side, side, 8), 2, cvb.LookupSpec(4, 4))
        recs += H.run_bench(sc, samplers=("dense",))
    lines = H.bench_csv(recs).strip().split("\n")
    assert lines[0] == "# corrvol-bench-csv v1"
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[1:]))))
    pos = [int(r["block_positions"]) for r in rows if r["sampler"] == "dense"]
    assert pos[1] / pos[0] == 16.0 and pos[2] / pos[1] == 16.0
    assert all(r["backend"] == "cuda" for r in rows)


@pytest.mark.gpu
def test_bench_counters_match_reference(cuda):
    """Block-store counters of the GPU sparse row equal the reference's."""
    ref = import_reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from corrvol.harness import gen_scenario as ref_gen, run_bench as ref_bench

    args = (7, (24, 40, 8), 5)
    ours = H.run_bench(cvb.gen_scenario(*args, cvb.LookupSpec(4, 3)), samplers=("sparse",),
                       block_sizes=(2, 4), cache_modes=(True, False))
    theirs = ref_bench(ref_gen(*args, ref.LookupSpec(4, 3)), samplers=("sparse",),
                       block_sizes=(2, 4), cache_modes=(True, False), backend="cython")
    for a, b in zip(ours, theirs):
        for f in ("dot_products", "macs", "blocks_computed", "blocks_stored", "blocks_union",
                  "block_positions"):
            assert getattr(a, f) == getattr(b, f), (f, a.block, a.cache)


def test_scenario_generator_matches_reference():
    """scenario.gen_scenario restates harness.gen_scenario (harness.py:66-127)
    bit for bit, so GPU and reference counters are compared on one input."""
    ref = import_reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from corrvol.harness import gen_scenario as ref_gen

    for seed, dims, n in [(3, (32, 32, 8), 6), (7, (24, 40, 8), 5), (0, (46, 62, 16), 3)]:
        a = cvb.gen_scenario(seed, dims, n, cvb.LookupSpec(4, 2))
        b = ref_gen(seed, dims, n, ref.LookupSpec(4, 2))
        assert np.array_equal(a.f1, b.f1.values) and np.array_equal(a.f2, b.f2.values)
        for ca, cb in zip(a.centroid_fields, b.centroid_fields):
            assert np.array_equal(ca, cb.coords)
