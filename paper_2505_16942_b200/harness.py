"""GPU benchmark / equivalence harness with the reference's records and CSV
schemas (mirrors corrvol/harness.py:190-540).

`run_bench` and `run_equivalence` drive this package's CUDA samplers on a
`SyntheticScenario` and return the reference's `BenchRecord` /
`EquivalenceReport` shapes, so the reference's counter-based acceptance
criteria (05 memory exponent, 06 caching, 07 work bound, 10 dense growth,
`test_acceptance.py:231-366`) can be re-asserted on GPU counters, and
`bench_csv` / `equivalence_csv` emit the reference's versioned CSV
(`# corrvol-bench-csv v1`, `# corrvol-verify-csv v1`) with backend=cuda.

"sparse" is the reference block-store pipeline (mode="block": its block
counters are bit-exact with the reference); "partial" is the B200 tile-cache
path (counters are cell dots).  wall_ms is device time (CUDA events).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import torch

from .dense import build_feature_pyramid, build_volume_pyramid, estimate_dense_bytes, lookup_dense
from .dense import pooled_dims
from .ondemand import lookup_on_demand
from .sparse import init_state, memory_footprint, sample_iteration
from .types import CentroidField, FeatureMap, WorkCounter

SAMPLERS = ("dense", "ondemand", "sparse", "partial")
DEFAULT_DENSE_LIMIT_BYTES = 2 * 2 ** 30  # harness.py:37


@dataclass
class BenchRecord:
    """One benchmark row (harness.py:278-301)."""

    sampler: str
    backend: str
    height: int
    width: int
    feature_dim: int
    radius: int
    levels: int
    block: int
    iterations: int
    cache: str
    seed: int
    dot_products: int
    macs: int
    blocks_computed: int
    blocks_stored: int
    blocks_union: int
    block_positions: int
    peak_bytes: int
    wall_ms: float
    shares: Optional[Dict[str, float]]
    oom: bool


class _Scn:
    """Scenario tensors on the GPU (fp32 features, centroid fields)."""

    def __init__(self, sc, device=None):
        dev = device if device is not None else torch.device("cuda")
        self.sc = sc
        self.spec = sc.spec
        self.f1 = FeatureMap(torch.from_numpy(sc.f1).to(dev), check=False)
        self.f2 = FeatureMap(torch.from_numpy(sc.f2).to(dev), check=False)
        self.cents = [CentroidField(torch.from_numpy(c).to(dev), check=False)
                      for c in sc.centroid_fields]


def _timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = fn()
    e1.record()
    torch.cuda.synchronize()
    return res, e0.elapsed_time(e1)


def _common(s: _Scn, sampler: str, block: int, cache: str) -> Dict:
    sc = s.sc
    return dict(sampler=sampler, backend="cuda", height=sc.height, width=sc.width,
                feature_dim=sc.feature_dim, radius=s.spec.radius, levels=s.spec.levels,
                block=block, iterations=sc.iterations, cache=cache, seed=sc.seed)


def _bench_dense(s: _Scn, dense_limit_bytes: int, strict: bool) -> BenchRecord:
    src = (s.sc.height, s.sc.width)
    est = estimate_dense_bytes(src, src, s.spec.levels)
    positions = sum(src[0] * src[1] * pooled_dims(src, l)[0] * pooled_dims(src, l)[1]
                    for l in range(s.spec.levels))
    common = _common(s, "dense", 1, "")
    common.update(blocks_computed=0, blocks_stored=0, blocks_union=0, block_positions=positions,
                  shares=None)
    if est > dense_limit_bytes:
        return BenchRecord(dot_products=0, macs=0, peak_bytes=est, wall_ms=0.0, oom=True,
                           **common)
    counter = WorkCounter()

    def run():
        vol = build_volume_pyramid(s.f1, s.f2, s.spec.levels, mode="pool_features",
                                   counter=counter, strict=strict)
        for c in s.cents:
            lookup_dense(vol, c, s.spec, strict=strict)
        return vol

    vol, ms = _timed(run)
    peak = vol.nbytes() + s.f1.values.numel() * 4 + s.f2.values.numel() * 4
    return BenchRecord(dot_products=counter.dot_products, macs=counter.macs, peak_bytes=peak,
                       wall_ms=ms, oom=False, **common)


def _bench_ondemand(s: _Scn, strict: bool) -> BenchRecord:
    counter = WorkCounter()

    def run():
        pyr = build_feature_pyramid(s.f2, s.spec.levels)
        for c in s.cents:
            lookup_on_demand(s.f1, pyr, c, s.spec, counter=counter, strict=strict)
        return pyr

    pyr, ms = _timed(run)
    peak = s.f1.values.numel() * 4 + sum(f.values.numel() * 4 for f in pyr.levels)
    common = _common(s, "ondemand", 1, "")
    return BenchRecord(dot_products=counter.dot_products, macs=counter.macs, blocks_computed=0,
                       blocks_stored=0, blocks_union=0, block_positions=0, peak_bytes=peak,
                       wall_ms=ms, shares=None, oom=False, **common)


def _bench_sparse(s: _Scn, block: int, cache_enabled: bool, strict: bool,
                  cache_cap_bytes: Optional[int], mode: str) -> BenchRecord:
    peaks = []

    def run():
        st = init_state(s.f1, s.f2, s.spec, block, cache_cap_bytes=cache_cap_bytes,
                        cache_enabled=cache_enabled, mode=mode, strict=strict)
        peaks.append(memory_footprint(st)["total_bytes"])
        for c in s.cents:
            sample_iteration(st, c)
            peaks.append(memory_footprint(st)["total_bytes"])
        return st

    st, ms = _timed(run)
    cnt = st.counter
    if mode == "block":
        stored = sum(lv.store.used for lv in st.levels)
        union = sum(int(lv.mask_union.sum().item()) for lv in st.levels)
        positions = sum(lv.block_positions for lv in st.levels)
    else:
        stored = union = positions = 0
    common = _common(s, "sparse" if mode == "block" else "partial", block,
                     "on" if cache_enabled else "off")
    return BenchRecord(dot_products=cnt.dot_products, macs=cnt.macs,
                       blocks_computed=cnt.blocks_computed if mode == "block" else 0,
                       blocks_stored=stored,
                       blocks_union=union, block_positions=positions, peak_bytes=max(peaks),
                       wall_ms=ms, shares=None, oom=False, **common)


def run_bench(scenario, samplers: Sequence[str] = ("dense", "ondemand", "sparse"),
              block_sizes: Sequence[int] = (4,), cache_modes: Sequence[bool] = (True,),
              dense_limit_bytes: int = DEFAULT_DENSE_LIMIT_BYTES,
              cache_cap_bytes: Optional[int] = None, strict: bool = True,
              device=None) -> List[BenchRecord]:
    """Benchmark samplers on one scenario (harness.py:440-472): dense and
    ondemand contribute one row each, sparse/partial one row per (block,
    cache mode).  Deterministic in every field except wall_ms."""
    s = _Scn(scenario, device)
    records = []
    for sampler in samplers:
        if sampler == "dense":
            records.append(_bench_dense(s, dense_limit_bytes, strict))
        elif sampler == "ondemand":
            records.append(_bench_ondemand(s, strict))
        elif sampler in ("sparse", "partial"):
            mode = "block" if sampler == "sparse" else "tile"
            for b in block_sizes:
                for cache in cache_modes:
                    records.append(_bench_sparse(s, b, cache, strict if mode == "block" else
                                                 strict, cache_cap_bytes, mode))
        else:
            raise ValueError(f"unknown sampler {sampler!r}; expected one of {SAMPLERS}")
    return records


@dataclass
class EquivalenceReport:
    """Per-iteration deviations vs dense (harness.py:146-164)."""

    block: int
    tolerance: float
    iterations: int
    per_iteration: List[Dict]
    max_deviation: float
    bitwise_ondemand: bool
    bitwise_sparse: bool
    passed: bool


def run_equivalence(scenario, block: int, tolerance: float = 1e-5,
                    dense_limit_bytes: int = DEFAULT_DENSE_LIMIT_BYTES,
                    cache_cap_bytes: Optional[int] = None, strict: bool = True,
                    device=None) -> EquivalenceReport:
    """Three-sampler equivalence on the GPU (harness.py:190-274): deviations
    max|a-b| / (1 + max|dense|) against the volume-pooled dense build, bitwise
    flags against the feature-pooled build, new blocks per iteration from the
    block-store sparse state."""
    s = _Scn(scenario, device)
    spec = s.spec
    est = estimate_dense_bytes((s.sc.height, s.sc.width), (s.sc.height, s.sc.width),
                               spec.levels)
    if est > dense_limit_bytes:
        raise ValueError(f"dense oracle would need {est} bytes (> limit {dense_limit_bytes}); "
                         "shrink dims or raise dense_limit_bytes")
    vol_default = build_volume_pyramid(s.f1, s.f2, spec.levels, mode="pool_volume",
                                       strict=strict)
    vol_matched = build_volume_pyramid(s.f1, s.f2, spec.levels, mode="pool_features",
                                       strict=strict)
    pyr = build_feature_pyramid(s.f2, spec.levels)
    state = init_state(s.f1, s.f2, spec, block, cache_cap_bytes=cache_cap_bytes, mode="block",
                       strict=strict)
    rows, max_dev, bit_od_all, bit_sp_all, prev = [], 0.0, True, True, 0
    for it, c in enumerate(s.cents):
        cd = lookup_dense(vol_default, c, spec, strict=strict).values
        cm = lookup_dense(vol_matched, c, spec, strict=strict).values
        co = lookup_on_demand(s.f1, pyr, c, spec, strict=strict).values
        cs = sample_iteration(state, c).values
        denom = 1.0 + float(cd.abs().max().item())
        d_do = float((co - cd).abs().max().item()) / denom
        d_ds = float((cs - cd).abs().max().item()) / denom
        d_os = float((cs - co).abs().max().item()) / denom
        bit_od = bool(torch.equal(co, cm))
        bit_sp = bool(torch.equal(cs, cm))
        bit_od_all &= bit_od
        bit_sp_all &= bit_sp
        blocks = state.counter.blocks_computed
        rows.append({"iteration": it, "dev_dense_ondemand": d_do, "dev_dense_sparse": d_ds,
                     "dev_ondemand_sparse": d_os, "bitwise_ondemand": bit_od,
                     "bitwise_sparse": bit_sp, "new_blocks": blocks - prev})
        prev = blocks
        max_dev = max(max_dev, d_do, d_ds, d_os)
    return EquivalenceReport(block=block, tolerance=tolerance, iterations=len(s.cents),
                             per_iteration=rows, max_deviation=max_dev,
                             bitwise_ondemand=bit_od_all, bitwise_sparse=bit_sp_all,
                             passed=max_dev <= tolerance)


VERIFY_CSV_SCHEMA = "# corrvol-verify-csv v1"
BENCH_CSV_SCHEMA = "# corrvol-bench-csv v1"
_BENCH_COLUMNS = (
    "sampler,backend,height,width,feature_dim,radius,levels,block,iterations,cache,seed,"
    "dot_products,macs,blocks_computed,blocks_stored,blocks_union,block_positions,"
    "peak_bytes,wall_ms,share_mask,share_indices,share_mmm,share_cache,share_sampling,oom"
)


def equivalence_csv(report: EquivalenceReport) -> str:
    """harness.py:478-492."""
    lines = [VERIFY_CSV_SCHEMA,
             "iteration,dev_dense_ondemand,dev_dense_sparse,dev_ondemand_sparse,"
             "bitwise_ondemand,bitwise_sparse,new_blocks"]
    for r in report.per_iteration:
        lines.append(f"{r['iteration']},{r['dev_dense_ondemand']:.6e},{r['dev_dense_sparse']:.6e},"
                     f"{r['dev_ondemand_sparse']:.6e},{int(r['bitwise_ondemand'])},"
                     f"{int(r['bitwise_sparse'])},{r['new_blocks']}")
    return "\n".join(lines) + "\n"


def bench_csv(records: Sequence[BenchRecord]) -> str:
    """harness.py:503-540, same columns and formatting."""
    lines = [BENCH_CSV_SCHEMA, _BENCH_COLUMNS]
    for r in records:
        shares = ["", "", "", "", ""] if r.shares is None else \
            [f"{r.shares[k]:.4f}" for k in ("mask", "indices", "mmm", "cache", "sampling")]
        lines.append(",".join(
            [r.sampler, r.backend, str(r.height), str(r.width), str(r.feature_dim),
             str(r.radius), str(r.levels), str(r.block), str(r.iterations), r.cache,
             str(r.seed), str(r.dot_products), str(r.macs), str(r.blocks_computed),
             str(r.blocks_stored), str(r.blocks_union), str(r.block_positions),
             str(r.peak_bytes), f"{r.wall_ms:.3f}"] + shares + ["1" if r.oom else "0"]))
    return "\n".join(lines) + "\n"
