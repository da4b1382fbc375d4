#!/usr/bin/env python
"""bench.py — corr-lookup ms/iter + peak HBM at 8K (L=4, r=4, D=256) vs roofline.

One step = one full lookup run of an image pair through the partial sampler:
fmap2 pyramid + init_state + 12 per-iteration `__call__(coords)` lookups
(BASELINE.json config 4: 540x960 features, D=256, L=4, r=4, 12 iterations).
Inputs are resident in HBM for `value`; `e2e` repeats the step through the
public API from pinned host buffers with every H2D/D2H inside the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {b200,reference}]
    torchrun --nproc-per-node N bench.py --gpus N ...   (query-row bands)

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import shutil
import tempfile
import time
from pathlib import Path
from typing import Optional

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# name: (H, W, D, radius, levels, iterations, normalize)
CONFIGS = {
    "C1": (46, 62, 256, 4, 4, 12, False),
    "C2": (135, 240, 256, 4, 4, 32, False),
    "C3": (270, 480, 256, 4, 4, 12, True),
    "C4": (540, 960, 256, 4, 4, 12, False),
    "C5": (270, 480, 256, 4, 4, 12, True),   # per pair; --batch pairs (seeds 0..B-1)
}
METRIC = "corr-lookup ms/iter + peak HBM at 8K (L=4,r=4,D=256) at 1/2/4/8 B200 vs roofline"
FP32_LANES_PER_SM = 128
N_SMS = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="C4")
    ap.add_argument("--variant", choices=["partial", "ondemand", "dense"], default="partial")
    ap.add_argument("--strict", action="store_true", help="reference-exact arithmetic")
    ap.add_argument("--batch", type=int, default=8, help="C5: image pairs in the batch")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch every kernel from the host each step instead of replaying "
                         "the step's captured CUDA graph")
    ap.add_argument("--gather", action="store_true",
                    help="C5 at N>1: all-gather every pair's costs to every rank per iteration")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-compare", action="store_true")
    ap.add_argument("--profile-only", action="store_true",
                    help="run warmup+steps only (for ncu); print nothing else")
    ap.add_argument("--cpu-baseline-worker", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--parity-dir", default=None, help=argparse.SUPPRESS)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the unmodified corrvol package, cython lane)
# ---------------------------------------------------------------------------

_REF_SC = None


def _ref_band_job(args):
    """Reference partial sampler (B=8) on rows [a, b) of the scenario; returns
    (t_prep_s, t_iters_s).  Runs in a forked worker, single-threaded."""
    a, b = args
    cv, sc = _REF_SC
    f1 = cv.FeatureMap(values=sc.f1[a:b])
    f2 = cv.FeatureMap(values=sc.f2)
    t0 = time.perf_counter()
    st = cv.init_state(f1, f2, cv.LookupSpec(*sc.spec_args), 8, backend="cython")
    t1 = time.perf_counter()
    for c in sc.centroid_fields:
        cv.sample_iteration(st, cv.CentroidField(coords=c[a:b].astype(np.float64)))
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


class _RefScenario:
    def __init__(self, cfg):
        from paper_2505_16942_b200.scenario import gen_scenario
        from paper_2505_16942_b200.types import LookupSpec

        h, w, d, r, levels, n_iter, norm = CONFIGS[cfg]
        sc = gen_scenario(0, (h, w, d), n_iter, LookupSpec(r, levels, norm),
                          coords_dtype=np.float32)
        self.f1, self.f2, self.centroid_fields = sc.f1, sc.f2, sc.centroid_fields
        self.spec_args = (r, levels, norm)
        self.h, self.w, self.iters = h, w, n_iter


def init_dist(torch, dist):
    """One process per GPU (torchrun env).  NCCL by default; CVB_BENCH_BACKEND=gloo
    exercises the multi-rank path with several ranks sharing one GPU (the
    scalar reductions then run on the host)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = os.environ.get("CVB_BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return world, rank, dev, (dev if backend == "nccl" else torch.device("cpu"))


def scenario_tensors(torch, dist, world, rank, red_dev, h, w, d, n_iter, spec, seed=0):
    """(f1 [H,W,D], f2 [H,W,D], coords [N,H,W,2] f32) as host tensors on every
    rank: generated once on rank 0 (gen_scenario recipe, fp32 centroids) and
    broadcast from it."""
    if rank == 0:
        import paper_2505_16942_b200 as cvb

        sc = cvb.gen_scenario(seed, (h, w, d), n_iter, spec, coords_dtype=np.float32)
        f1 = torch.from_numpy(sc.f1)
        f2 = torch.from_numpy(sc.f2)
        co = torch.from_numpy(np.stack(sc.centroid_fields))
    else:
        f1 = torch.empty((h, w, d), dtype=torch.float32)
        f2 = torch.empty((h, w, d), dtype=torch.float32)
        co = torch.empty((n_iter, h, w, 2), dtype=torch.float32)
    if world > 1:
        out = []
        for t in (f1, f2, co):
            buf = t.to(red_dev)
            dist.broadcast(buf, src=0)
            out.append(buf.cpu() if buf.is_cuda else buf)
        f1, f2, co = out
    return f1, f2, co


def reference_sample(cfg: str, workers: int, rows_per_worker: int):
    """Time the reference on `workers` parallel row bands; extrapolate to the frame.

    The reference hot path is single-threaded (numpy + GIL-held Cython,
    _ckernels.pyx:1), so the all-cores figure runs one process per core on
    disjoint row bands.  Frame time on `workers` cores =
    prep (fmap2 pyramid + patch-major, once per core) + per-band iteration time
    x frame_rows / (rows_per_worker * workers).
    """
    global _REF_SC
    from oracle import import_reference

    cv = import_reference()
    if cv is None:
        raise RuntimeError("oracle/_ref not built")
    if _REF_SC is None:
        _REF_SC = (cv, _RefScenario(cfg))
    sc = _REF_SC[1]
    # disjoint bands spread over the frame, starting at multiples of 8 rows
    # (the last one may be shorter); with enough workers they cover the frame
    n_slots = max(1, -(-sc.h // rows_per_worker))
    workers = min(workers, n_slots)
    picks = sorted({int(round(i * (n_slots - 1) / max(1, workers - 1))) for i in range(workers)})
    if workers == 1:
        picks = [n_slots // 2]
    bands = [(p * rows_per_worker, min((p + 1) * rows_per_worker, sc.h)) for p in picks]
    workers = len(bands)
    t0 = time.perf_counter()
    if workers == 1:
        res = [_ref_band_job(bands[0])]
    else:
        ctx = mp.get_context("fork")
        with ctx.Pool(workers) as pool:
            res = pool.map(_ref_band_job, bands)
    wall = time.perf_counter() - t0
    prep = statistics.mean(r[0] for r in res)
    iters = statistics.mean(r[1] for r in res)
    rows_done = sum(b - a for a, b in bands)
    # bands covering the frame run concurrently: the frame takes the slowest
    # band; otherwise the frame needs h / rows_done rounds of the sampled bands
    frame_s = (prep + max(r[1] for r in res) if rows_done >= sc.h
               else prep + iters * sc.h / rows_done)
    return {"ms_per_iter": 1e3 * frame_s / sc.iters, "frame_s": frame_s, "wall_s": wall,
            "prep_s": prep, "iters_s_per_band": iters, "bands": bands, "cores": workers,
            "iterations": sc.iters}


def workload(cfg: str, batch: int = 0) -> str:
    """The `config.workload` string; identical in both arms."""
    h, w, d, r, levels, n_iter, norm = CONFIGS[cfg]
    pairs = f"batch of {batch} image pairs" if cfg == "C5" else "one image pair"
    return (f"{cfg} {h}x{w} features D={d} L={levels} r={r} {n_iter} iterations"
            f"{' normalize' if norm else ''}, {pairs} per step")


def host_info() -> dict:
    """Host cores the CPU legs can use (nproc) plus the lscpu model line."""
    info = {"nproc": os.cpu_count(), "affinity_cores": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k.strip()] = v.strip()
    except Exception:
        pass
    return info


PARITY_ROWS = 16  # rows of the timed reference band checked against the GPU


def _partial_band(cfg: str):
    """Rows the CPU-baseline worker times the reference partial sampler on:
    the whole frame at C1, else a 32-row band of whole tiles mid-frame."""
    h = CONFIGS[cfg][0]
    if cfg == "C1":
        return 0, h
    a = h // 2 // 8 * 8
    return a, a + 32


def _ref_variant_times(cfg: str, parity_dir: Optional[str] = None) -> dict:
    """The reference's three samplers on ONE core (harness.py:304-437):
    full runs at C1; at larger configs the partial sampler on a 32-row band
    (all iterations) and on-demand on an 8-row band (first 2 iterations), both
    extrapolated linearly in rows (and iterations); dense is reported
    infeasible when its volume exceeds the reference bench's dense limit
    (DEFAULT_DENSE_LIMIT_BYTES = 2 GiB, harness.py:33,330-333)."""
    from oracle import import_reference

    cv = import_reference()
    if cv is None:
        raise RuntimeError("oracle/_ref not built")
    h, w, d, r, levels, n_iter, norm = CONFIGS[cfg]
    sc = _RefScenario(cfg)
    spec = cv.LookupSpec(r, levels, norm)
    cents = [c.astype(np.float64) for c in sc.centroid_fields]
    full = cfg == "C1"
    res = {}
    # partial
    a, b = _partial_band(cfg)
    f1 = cv.FeatureMap(values=sc.f1[a:b])
    f2 = cv.FeatureMap(values=sc.f2)
    # the GPU's outputs for the first PARITY_ROWS rows of this band (fast and
    # strict arithmetic, every iteration), written by the B200 arm: the
    # reference's own outputs check them here, outside the timed calls
    fast = strict = None
    if parity_dir is not None:
        fast = np.load(os.path.join(parity_dir, "fast.npy"), mmap_mode="r")
        strict = np.load(os.path.join(parity_dir, "strict.npy"), mmap_mode="r")
    pr = min(PARITY_ROWS, b - a)
    n1 = float(np.sqrt((sc.f1[a:a + pr].astype(np.float64) ** 2).sum(-1)).max())
    n2 = float(np.sqrt((sc.f2.astype(np.float64) ** 2).sum(-1)).max())
    dev = ns = 0.0
    bitwise = True
    t0 = time.perf_counter()
    st = cv.init_state(f1, f2, spec, 8, backend="cython")
    t1 = time.perf_counter()
    t_it = 0.0
    for i, c in enumerate(cents):
        tq = time.perf_counter()
        cm = cv.sample_iteration(st, cv.CentroidField(coords=c[a:b]))
        t_it += time.perf_counter() - tq
        if fast is not None:
            want = np.asarray(cm.values)[:pr]
            d = float(np.abs(np.asarray(fast[i]) - want).max())
            dev = max(dev, d / (1.0 + float(np.abs(want).max())))
            ns = max(ns, d / max(n1 * n2, 1e-30))
            bitwise = bitwise and np.array_equal(np.asarray(strict[i]), want)
    t2 = time.perf_counter()
    frame_s = (t1 - t0) + t_it * h / (b - a)
    res["partial"] = {"ms_per_iter": 1e3 * frame_s / n_iter, "rows": [a, b],
                      "iterations": n_iter, "measured_s": (t1 - t0) + t_it,
                      "extrapolated": not full}
    if fast is not None:
        res["parity"] = {"checker": "reference corrvol 0.1.0 partial sampler (the timed band)",
                         "rows": [a, a + pr], "iterations": n_iter,
                         "fast_ref_gate": dev, "fast_ns_gate": ns,
                         "strict_bitwise": bool(bitwise),
                         "gates": {"ref": 1e-5, "ns": 1e-4},
                         "pass": bool(bitwise and dev <= 1e-5 and ns <= 1e-4)}
    # on-demand
    a, b = (0, h) if full else (h // 2 // 8 * 8, h // 2 // 8 * 8 + 8)
    its = n_iter if full else 2
    f1 = cv.FeatureMap(values=sc.f1[a:b])
    t0 = time.perf_counter()
    pyr = cv.build_feature_pyramid(f2, levels)
    t1 = time.perf_counter()
    for c in cents[:its]:
        cv.lookup_on_demand(f1, pyr, cv.CentroidField(coords=c[a:b]), spec, backend="cython")
    t2 = time.perf_counter()
    frame_s = (t1 - t0) + (t2 - t1) * (h / (b - a)) * (n_iter / its)
    res["ondemand"] = {"ms_per_iter": 1e3 * frame_s / n_iter, "rows": [a, b],
                       "iterations": its, "measured_s": t2 - t0, "extrapolated": not full}
    # dense (pool_features build + lookups, the bench's mode, harness.py:336-338)
    est = cv.estimate_dense_bytes((h, w), (h, w), levels)
    limit = 2 * 2 ** 30
    if est > limit:
        res["dense"] = {"oom": True, "bytes": est, "limit_bytes": limit,
                        "note": "infeasible: reported as harness.py:330-333 reports it"}
    else:
        f1 = cv.FeatureMap(values=sc.f1)
        t0 = time.perf_counter()
        vol = cv.build_volume_pyramid(f1, f2, levels, mode="pool_features", backend="cython")
        t1 = time.perf_counter()
        for c in cents:
            cv.lookup_dense(vol, cv.CentroidField(coords=c), spec)
        t2 = time.perf_counter()
        res["dense"] = {"ms_per_iter": 1e3 * (t2 - t0) / n_iter, "build_s": t1 - t0,
                        "iterations": n_iter, "measured_s": t2 - t0, "extrapolated": False}
    return res


def cpu_baseline_worker(cfg: str, parity_dir: Optional[str] = None) -> None:
    print(json.dumps(_ref_variant_times(cfg, parity_dir)))


def _ref_cores(cfg: str) -> int:
    """Worker processes for the reference arm: every host core, bounded by host
    memory (each worker holds the fmap2 pyramid and its patch-major copies,
    about 3x fmap2's bytes) and by the frame's 8-row bands."""
    h, w, d = CONFIGS[cfg][:3]
    cores = min(len(os.sched_getaffinity(0)), -(-h // 8))
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
        cores = max(1, min(cores, int(avail * 0.6 // (3 * h * w * d * 4))))
    except (ValueError, OSError):
        cores = min(cores, 16)
    return cores


def run_reference_arm(args) -> None:
    """The reference's own CPU partial sampler on all usable host cores.

    One step = one bounded sample of the workload: every worker runs the
    reference (init_state + all iterations) on its own 8-row band of the
    frame, disjoint bands spread over the frame.  `ms_per_step` is the
    measured wall time of that sample; `value` (ms per lookup iteration of the
    whole frame) scales the per-band iteration time by frame rows / sampled
    rows — `extrapolation` says by how much (1.0 when the bands cover the
    frame)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = "C3" if args.config == "C5" else args.config
    cores = _ref_cores(cfg)
    h, w, d, r, levels, n_iter, norm = CONFIGS[cfg]
    vals, walls = [], []
    res = None
    for i in range(args.warmup + args.steps):
        res = reference_sample(cfg, cores, 8)
        cores = res["cores"]
        if i >= args.warmup:
            vals.append(res["ms_per_iter"])
            walls.append(res["wall_s"])
    rows_done = sum(b - a for a, b in res["bands"])
    v = statistics.mean(vals) * (args.batch if args.config == "C5" else 1)
    sample = (f"reference corrvol 0.1.0 partial sampler (B=8, cython lane), {cores} processes x "
              f"one 8-row band each ({rows_done} of {h} rows of {cfg}), all {n_iter} iterations "
              f"per band; value = per-band iteration time x {h}/{rows_done} rows"
              + (f" x {args.batch} pairs" if args.config == "C5" else ""))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "ms/iter",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.mean(walls), 3), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload(args.config, args.batch),
                   "parallelism": f"{cores} CPU processes"},
        "extrapolation": {"sampled_rows": rows_done, "frame_rows": h,
                          "factor": round(h / rows_done, 4)},
        "host": host_info(),
        "cpu_baseline": {"value": round(v, 3), "unit": "ms/iter", "cores": cores,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(v, 3), "unit": "ms/iter", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _parity_outputs(cvb, torch, f1_dev, f2_dev, cents, spec, cfg: str, pdir: str) -> None:
    """The GPU's cost maps on the rows the CPU-baseline worker's reference band
    starts with (_partial_band): fast arithmetic from a full-frame sampler,
    strict from a sampler on the band's rows (row bands of whole 8-row tiles
    are exact), every iteration; saved for the worker to check."""
    a, ref_b = _partial_band(cfg)
    b = min(ref_b, a + PARITY_ROWS)
    fast = cvb.CorrSampler(cvb.FeatureMap(f1_dev, check=False), cvb.FeatureMap(f2_dev, check=False),
                           spec, check=False)
    strict = cvb.CorrSampler(cvb.FeatureMap(f1_dev[a:ref_b].contiguous(), check=False),
                             cvb.FeatureMap(f2_dev, check=False), spec, strict=True, check=False)
    got_f, got_s = [], []
    for c in cents:
        got_f.append(fast(c).values[a:b].cpu().numpy())
        band = cvb.CentroidField(c.coords[a:ref_b].contiguous(), check=False)
        got_s.append(strict(band).values[:b - a].cpu().numpy())
    np.save(os.path.join(pdir, "fast.npy"), np.stack(got_f))
    np.save(os.path.join(pdir, "strict.npy"), np.stack(got_s))
    del fast, strict
    torch.cuda.empty_cache()


def cpu_baseline(cfg: str, parity_dir: Optional[str] = None) -> dict:
    """`cpu_baseline` of the B200 arm: the reference's dense, on-demand and
    partial samplers timed on ONE host core (taskset -c 0) in a subprocess;
    `value` is the partial sampler (the path this build replaces).  With
    `parity_dir` the reference's partial outputs also check the GPU's on the
    first rows of its band (returned under "parity", popped by the caller)."""
    try:
        cmd = ["taskset", "-c", "0", sys.executable, str(ROOT / "bench.py"),
               "--cpu-baseline-worker", cfg]
        if parity_dir is not None:
            cmd += ["--parity-dir", parity_dir]
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        ref = json.loads(res.stdout.strip().splitlines()[-1])
        parity = ref.pop("parity", None)
        p = ref["partial"]
        parts = []
        for name in ("partial", "ondemand", "dense"):
            v = ref[name]
            if v.get("oom"):
                parts.append(f"dense infeasible ({v['bytes'] / 1e9:.1f} GB volume)")
            else:
                how = (f"rows {v['rows'][0]}..{v['rows'][1]}, {v['iterations']} iterations, "
                       "extrapolated" if v.get("extrapolated") else "full frame, all iterations")
                parts.append(f"{name} {v['ms_per_iter']:.1f} ms/iter ({how})")
        return {"value": round(p["ms_per_iter"], 3), "unit": "ms/iter", "cores": 1,
                "kind": "reference",
                "sample": f"reference corrvol 0.1.0 (cython lane), 1 core (taskset -c 0), "
                          f"{cfg}: " + "; ".join(parts),
                "variants": {k: {kk: (round(vv, 3) if isinstance(vv, float) else vv)
                                 for kk, vv in v.items()} for k, v in ref.items()},
                "host": host_info(), "parity": parity}
    except Exception as exc:  # report, never fake
        return {"value": None, "unit": "ms/iter", "cores": 1, "kind": "reference",
                "sample": f"failed: {type(exc).__name__}: {exc}"[:300]}


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------

class Clocks:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.file = None

    def start(self):
        try:
            self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.file, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.file.flush()
        rows = [l.split(",") for l in Path(self.file.name).read_text().splitlines() if l.strip()]
        os.unlink(self.file.name)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for row in rows:
            try:
                smax = float(row[2])
                if float(row[1]) < 0.3 * smax:  # idle sample (before the first launch)
                    continue
                sm.append(float(row[1]))
                for nm, v in zip(names, row[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def main():
    args = parse()
    if args.cpu_baseline_worker:
        cpu_baseline_worker(args.cpu_baseline_worker, args.parity_dir)
        return
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.config == "C5":
        run_batch(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2505_16942_b200 as cvb
    from paper_2505_16942_b200 import _lib
    from paper_2505_16942_b200.parallel import row_bands
    from paper_2505_16942_b200.sparse import sample_iteration_timed

    world, rank, dev, red_dev = init_dist(torch, dist)

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    h, w, d, r, levels, n_iter, norm = CONFIGS[args.config]
    spec = cvb.LookupSpec(r, levels, norm)
    # rank 0 generates the pair; fmap2 (replicated) and the fmap1 / centroid
    # rows are broadcast to the other ranks (NCCL over NVLink, or gloo on the
    # host), each rank keeping its query-row band
    f1_all, f2_all, co_all = scenario_tensors(torch, dist, world, rank, red_dev, h, w, d, n_iter,
                                              spec)
    a, b = row_bands(h, world)[rank]
    rows = b - a
    f1_host = f1_all[a:b].contiguous()
    f2_host = f2_all
    co_host = [co_all[i, a:b].contiguous() for i in range(n_iter)]
    del f1_all, co_all
    f1_dev = f1_host.to(dev)
    f2_dev = f2_host.to(dev)
    co_dev = [c.to(dev) for c in co_host]
    k1 = spec.window
    out = torch.empty((rows, w, levels, k1, k1), dtype=torch.float32, device=dev)
    cents = [cvb.CentroidField(c, check=False) for c in co_dev]

    def step(variant=args.variant, cache=True):
        s = cvb.CorrSampler(cvb.FeatureMap(f1_dev, check=False),
                            cvb.FeatureMap(f2_dev, check=False), spec, variant=variant,
                            strict=args.strict, cache=cache, check=False)
        for c in cents:
            s(c, out=out)
        return s

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        return allmax(e0.elapsed_time(e1) / steps)

    main_step = step
    graph_launches = 0
    # peak HBM covers the whole step's allocations, including the buffers a
    # CUDA graph keeps in its private pool from capture time on
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    base_alloc = torch.cuda.memory_allocated(dev)
    if args.graph:
        # the whole step (prepare + every lookup) captured once into a CUDA graph
        # over the static input/output buffers and replayed (no per-launch host
        # cost; matters for launch-bound frames such as C1)
        step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        n0 = _lib.launch_count()
        with torch.cuda.graph(graph):
            step()
        graph_launches = _lib.launch_count() - n0
        main_step = graph.replay

    if args.profile_only:
        timed(main_step, args.steps, args.warmup)
        return

    # ---- main measurement: inputs resident in HBM -------------------------
    # nvidia-smi samples clocks from before the warm-up to the end of the timed
    # region (the GPU is under load the whole time); it needs ~1 s to start.
    clocks = Clocks(dev.index).start()
    time.sleep(1.5)
    for _ in range(args.warmup):
        main_step()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    ms_step = timed(main_step, args.steps, 0)
    launches = _lib.launch_count() - launches0 + graph_launches * args.steps
    clk = clocks.stop()
    peak_bytes = int(allmax(torch.cuda.max_memory_allocated(dev)))
    ms_iter = ms_step / n_iter
    p_total = h * w
    lookups_s = p_total * n_iter / (ms_step / 1e3)

    # ---- per-kernel timing (tile mode): contraction vs gather/sampler -----
    kern = {}
    if args.variant == "partial":
        st = cvb.init_state(cvb.FeatureMap(f1_dev, check=False), cvb.FeatureMap(f2_dev, check=False),
                            spec, strict=args.strict)
        evs = [sample_iteration_timed(st, c, out) for c in cents]
        torch.cuda.synchronize()
        t_con = [e[0].elapsed_time(e[1]) for e in evs]
        t_gat = [e[1].elapsed_time(e[2]) for e in evs]
        kern = {"contract_ms": t_con, "gather_ms": t_gat,
                "device_counters": st.device_counters, "tensor_cores": st.tc}
        del st

    # ---- roofline ----------------------------------------------------------
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    peaks = json.loads(peaks_path.read_text()) if peaks_path.exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "measured" if "hbm_gbs" in peaks else "fallback"
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    # dram bytes per launch from the committed `ncu --set full` capture (or null)
    traffic_path = ROOT / "profiles" / f"ncu_traffic_{args.config}.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    if rows != h:  # the capture is of a full-frame launch; this rank runs a row band
        traffic = {k: int(v * rows / h) for k, v in traffic.items() if isinstance(v, (int, float))}
    geom_path = ROOT / "profiles" / f"geometry_{args.config}.json"
    geom = json.loads(geom_path.read_text()) if geom_path.exists() else None
    out_bytes_iter = rows * w * levels * k1 * k1 * 4
    coord_bytes_iter = rows * w * 2 * 4
    roofline = None
    secondary = None
    if kern:
        tc, tg = sum(kern["contract_ms"]), sum(kern["gather_ms"])
        gather_bytes = (out_bytes_iter + coord_bytes_iter) * n_iter
        gather_gbs = gather_bytes / (tg / 1e3) / 1e9
        r_gather = {"kernel": "gather_fast_kernel (partial gather / bilinear sampler)", "bound": "hbm",
                    "achieved": round(gather_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(gather_gbs / hbm_peak, 4),
                    "traffic": traffic.get("gather_fast_kernel"),
                    "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({hbm_src})",
                    "alg_bytes_per_launch": gather_bytes / n_iter,
                    "avg_launch_ms": tg / n_iter, "share_of_step": round(tg / (tc + tg), 3)}
        fp32_peak = N_SMS * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
        r_con = None
        if geom is not None and world == 1:
            flops = geom["flops_alg_run"]
            tf = flops / (tc / 1e3) / 1e12
            if kern["tensor_cores"]:
                peak = peaks.get("bf16_tflops_sustained", 1400.0)
                src = ("MEASURED_PEAKS.json bf16_tflops_sustained (kind::f16 dense rate; "
                       "kernel timed inside the step)" if "bf16_tflops_sustained" in peaks
                       else "fallback 1.4 PFLOP/s sustained")
                name = "partial_contract_tcp_kernel (tiler + incremental tcgen05 contraction)"
                bound = "tensor"
                executed = 3 * 2 * d * kern["device_counters"]["dots"]
            else:
                peak = fp32_peak
                src = ("FFMA nominal 148 SM x 128 lanes x 2 x sm_max_mhz "
                       "(no measured FP32 peak; MEASURED_PEAKS has HBM/bf16 only)")
                name = "partial_contract_kernel (tiler + incremental FFMA contraction)"
                bound = "fp32"
                executed = 2 * d * kern["device_counters"]["dots"]
            r_con = {"kernel": name, "bound": bound, "achieved": round(tf, 2),
                     "peak": round(peak, 1), "unit": "TFLOP/s", "frac": round(tf / peak, 4),
                     "traffic": traffic.get("partial_contract_tcp_kernel" if kern["tensor_cores"]
                                            else "partial_contract_kernel"),
                     "peak_source": src,
                     "alg_flops_per_launch": flops / n_iter, "avg_launch_ms": tc / n_iter,
                     "share_of_step": round(tc / (tc + tg), 3),
                     "executed_flops": executed,
                     "note": "achieved = algorithmic flops (2*D*compulsory union cells, "
                             "profiles/geometry_*.json) / measured contraction time"}
        # measured DRAM traffic of one warm launch (committed ncu capture) over
        # the warm launch time: how close each kernel runs to the HBM roofline
        for r_, warm_ms in ((r_gather, statistics.mean(kern["gather_ms"][1:])),
                            (r_con, statistics.mean(kern["contract_ms"][1:]))):
            if r_ is not None and r_.get("traffic"):
                gbs = r_["traffic"] / (warm_ms / 1e3) / 1e9
                r_["traffic_gbs_warm"] = round(gbs, 1)
                r_["traffic_frac_of_hbm_peak"] = round(gbs / hbm_peak, 4)
        if r_con is not None and tc >= tg:
            roofline, secondary = r_con, r_gather
        else:
            roofline, secondary = r_gather, r_con

    # ---- run-level roofline ---------------------------------
    pyr_bytes = sum((h >> l) * (w >> l) for l in range(1, levels)) * d * 4
    bytes_alg = n_iter * (out_bytes_iter + coord_bytes_iter) * world + h * w * d * 8 + 2 * pyr_bytes
    run_floor_ms = bytes_alg / (hbm_peak * 1e9) * 1e3

    # ---- comparisons in the same build (N=1) --------------------------------
    compare = {}
    dense_bytes = cvb.estimate_dense_bytes((h, w), (h, w), levels)
    if not args.no_compare and world == 1:
        compare["ondemand_ms_per_iter"] = round(timed(lambda: step("ondemand"), 1, 1) / n_iter, 3)

        def ondemand_literal():  # the reference algorithm's per-query window dots (FFMA)
            pyr = cvb.build_feature_pyramid(cvb.FeatureMap(f2_dev, check=False), levels)
            f1m = cvb.FeatureMap(f1_dev, check=False)
            for c in cents:
                cvb.lookup_on_demand(f1m, pyr, c, spec, out=out)

        compare["ondemand_per_query_ffma_ms_per_iter"] = round(
            timed(ondemand_literal, 1, 1) / n_iter, 3)
        compare["partial_nocache_ms_per_iter"] = round(
            timed(lambda: step("partial", cache=False), 1, 1) / n_iter, 3)
        torch.cuda.empty_cache()
        free, _ = torch.cuda.mem_get_info(dev)
        try:
            if dense_bytes >= 0.85 * free:
                raise MemoryError
            compare["dense_ms_per_iter"] = round(timed(lambda: step("dense"), 1, 1) / n_iter, 3)
        except (MemoryError, torch.cuda.OutOfMemoryError):
            # reported the way harness.py:330-333 reports a dense OOM
            torch.cuda.empty_cache()
            compare["dense"] = {"oom": True, "bytes": dense_bytes, "free_bytes": free}
    torch.cuda.synchronize()

    # ---- e2e: public API from pinned host buffers ---------------------------
    e2e = None
    if not args.no_e2e:
        f1_pin = f1_host.pin_memory()
        f2_pin = f2_host.pin_memory()
        co_pin = [c.pin_memory() for c in co_host]
        outs_pin = [torch.empty(out.shape, dtype=torch.float32).pin_memory() for _ in range(2)]
        # two download streams, one per output buffer: two copy engines keep
        # the D2H link fuller (56.4 vs 55.6 GB/s, profiles/r01/pcie_bw.txt)
        d2h_streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
        h2d_stream = torch.cuda.Stream(dev)

        def e2e_step():
            # inputs on their own copy stream (PCIe is full duplex: the next
            # step's uploads overlap this step's trailing downloads)
            main = torch.cuda.current_stream()
            with torch.cuda.stream(h2d_stream):
                f1d = f1_pin.to(dev, non_blocking=True)
                f2d = f2_pin.to(dev, non_blocking=True)
                cds = [c.to(dev, non_blocking=True) for c in co_pin]
                ev_in = torch.cuda.Event()
                ev_in.record(h2d_stream)
            main.wait_event(ev_in)
            for t in [f1d, f2d] + cds:
                t.record_stream(main)
            s = cvb.CorrSampler(cvb.FeatureMap(f1d, check=False), cvb.FeatureMap(f2d, check=False),
                                spec, variant=args.variant, strict=args.strict, check=False)
            bufs = [torch.empty_like(out), torch.empty_like(out)]
            done = [None, None]
            for i, c in enumerate(cds):
                j = i % 2
                if done[j] is not None:
                    main.wait_event(done[j])
                res = s(cvb.CentroidField(c, check=False), out=bufs[j])
                ev = torch.cuda.Event()
                ev.record(main)
                d2h = d2h_streams[j]
                with torch.cuda.stream(d2h):
                    d2h.wait_event(ev)
                    outs_pin[j].copy_(res.values, non_blocking=True)
                    done[j] = torch.cuda.Event()
                    done[j].record(d2h)
            for b_, d2h in zip(bufs, d2h_streams):
                b_.record_stream(d2h)
            for d2h in d2h_streams:
                main.wait_stream(d2h)

        e2e_steps = args.steps
        ms_e2e = timed(e2e_step, e2e_steps, 1)
        e2e = {"value": round(ms_e2e / n_iter, 3), "unit": "ms/iter",
               "h2d_bytes_per_step": (f1_host.numel() + f2_host.numel()) * 4 +
               sum(c.numel() * 4 for c in co_host),
               "d2h_bytes_per_step": out.numel() * 4 * n_iter,
               "steps": e2e_steps,
               "note": "CorrSampler from pinned host fmaps + coords (H2D copy stream), "
                       "every iteration's full cost map D2H to pinned host (double-buffered, "
                       "one download stream per buffer); PCIe-bound"}

    # ---- CPU baseline (rank 0, N=1) ----------------------------------------
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        pdir = None
        if args.variant == "partial" and not args.strict:
            pdir = tempfile.mkdtemp(prefix="cvb_parity_")
            _parity_outputs(cvb, torch, f1_dev, f2_dev, cents, spec, args.config, pdir)
        cpu = cpu_baseline(args.config, pdir)
        parity = cpu.pop("parity", None)
        if pdir is not None:
            shutil.rmtree(pdir, ignore_errors=True)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(ms_iter, 4), "unit": "ms/iter",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 3), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded N(0,1) fmaps, Gaussian-smoothed flow drift; "
                    "gen_scenario recipe, fp32 centroids)",
            "config": {"workload": workload(args.config),
                       "variant": args.variant, "arith": "strict" if args.strict else "fast",
                       "parallelism": f"query-row bands x{world}" if world > 1 else "1 GPU",
                       "cuda_graph": bool(args.graph),
                       "l2": "inputs larger than L2 (fmaps 2x531 MB, cache GBs)"},
            "lookups_per_s": round(lookups_s, 1),
            "peak_hbm_bytes": peak_bytes,
            "peak_hbm_bytes_over_inputs": peak_bytes - base_alloc if world == 1 else None,
            "dense_bytes": dense_bytes,
            "memory_reduction_vs_dense": round(1 - peak_bytes / dense_bytes, 5),
            "roofline": roofline, "roofline_secondary": secondary,
            "run_roofline": {"bytes_alg": bytes_alg, "floor_ms_per_step": round(run_floor_ms, 4),
                             "frac": round(run_floor_ms / ms_step, 4),
                             "flops_alg": geom["flops_alg_run"] if geom else None},
            "kernel_ms": {k: [round(x, 4) for x in v] for k, v in kern.items()
                          if k.endswith("_ms")} if kern else None,
            "tensor_cores": kern.get("tensor_cores") if kern else None,
            "device_counters": kern.get("device_counters") if kern else None,
            "compare": compare or None,
            "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "clocks": clk,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_batch(args) -> None:
    """C5: a batch of 4K pairs (SEA-RAFT sampler config, normalize=True) on
    ONE batched state per rank (one plan + contraction + sampler launch per
    iteration over every pair's tiles), batch slices per rank with no
    data-path collective; --gather adds the per-iteration all-gather of the
    sampled costs (timed separately).  The whole step (prepare + 12 lookups)
    is one captured CUDA graph, as for C1-C4.  Scenarios: seeds 0..7,
    reused cyclically beyond 8 pairs (generation is CPU-bound)."""
    import torch
    import torch.distributed as dist

    import paper_2505_16942_b200 as cvb
    from paper_2505_16942_b200 import _lib
    from paper_2505_16942_b200.parallel import batch_slices, gather_bands

    world, rank, dev, red_dev = init_dist(torch, dist)
    h, w, d, r, levels, n_iter, norm = CONFIGS["C5"]
    spec = cvb.LookupSpec(r, levels, norm)
    slices = batch_slices(args.batch, world)
    a, b = slices[rank]
    uniq = {}
    for s_ in range(a, b):
        if s_ % 8 not in uniq:
            uniq[s_ % 8] = cvb.gen_scenario(s_ % 8, (h, w, d), n_iter, spec,
                                            coords_dtype=np.float32)
    scs = [uniq[s_ % 8] for s_ in range(a, b)]
    f1 = torch.stack([torch.from_numpy(sc.f1) for sc in scs]).to(dev)
    f2 = torch.stack([torch.from_numpy(sc.f2) for sc in scs]).to(dev)
    coords = [torch.stack([torch.from_numpy(sc.centroid_fields[i]) for sc in scs]).to(dev)
              for i in range(n_iter)]
    k = spec.window
    out = torch.empty((b - a, h, w, levels, k, k), dtype=torch.float32, device=dev)
    t_gather = [0.0]

    def step():
        s = cvb.BatchCorrSampler(f1, f2, spec, strict=args.strict, graph=False)
        for c in coords:
            s(c, out=out)

    def single_step():
        s = cvb.CorrSampler(f1[0], f2[0], spec, strict=args.strict, check=False)
        for c in coords:
            s(c[0], out=out[0])

    def capture(fn):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        n0 = _lib.launch_count()
        with torch.cuda.graph(g):
            fn()
        return g, _lib.launch_count() - n0

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    graph, g_launches = capture(step)
    clocks = Clocks(dev.index).start()
    time.sleep(1.5)
    ms = timed(graph.replay, args.steps, args.warmup)
    clk = clocks.stop()
    peak = torch.cuda.max_memory_allocated(dev)
    del graph
    torch.cuda.empty_cache()
    g1, _ = capture(single_step)
    ms_single = timed(g1.replay, args.steps, args.warmup)
    del g1
    if args.gather and world > 1:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n_iter):
            gather_bands(out, slices)
        e1.record()
        e1.synchronize()
        t_gather[0] = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms, float(peak), ms_single], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, peak, ms_single = float(t[0]), int(t[1]), float(t[2])
        dist.barrier()
    if rank == 0:
        print(json.dumps({
            "metric": METRIC + " [C5 batch sweep]", "value": round(ms / n_iter, 4),
            "unit": "ms/iter", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (gen_scenario seeds 0..7, reused cyclically beyond 8 pairs)",
            "config": {"workload": workload("C5", args.batch),
                       "parallelism": f"batch slices x{world}", "cuda_graph": True,
                       "l2": "inputs larger than L2"},
            "pairs_per_rank": b - a,
            "single_pair_ms_per_iter": round(ms_single / n_iter, 4),
            "batch_vs_pairs_x_single": round(ms / ((b - a) * ms_single), 4),
            "lookups_per_s": round(args.batch * h * w * n_iter / (ms / 1e3), 1),
            "peak_hbm_bytes_per_gpu": peak,
            "allgather_ms_per_iter": round(t_gather[0] / n_iter, 3) if args.gather else None,
            "clocks": clk, "gpu_launches": g_launches * args.steps, "e2e": None}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
