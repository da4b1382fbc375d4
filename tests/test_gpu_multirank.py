"""The multi-rank product path on the GPU.

Ranks are separate processes (one per GPU in production); here 2 gloo ranks
share the box's one B200.  Each rank runs the CUDA sampler on its share of
the work — a query-row band of the frame (CorrSampler) or a slice of the
batch (BatchCorrSampler) — and `gather_bands` reassembles the frame.  The
reassembled output must equal the single-process run bit for bit (same
kernels, same per-query arithmetic; bands start on 8-row tile boundaries).
The bench's multi-rank launch (torchrun, barrier, max-over-ranks timing,
rank-0 line, fmap broadcast from rank 0) runs the same way.
"""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.multiprocessing as tmp

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        sys.path.insert(0, str(ROOT))
        import torch.distributed as dist

        import paper_2505_16942_b200 as cvb
        from paper_2505_16942_b200.parallel import batch_slices, gather_bands, row_bands

        dist.init_process_group("gloo", rank=rank, world_size=world)
        dev = torch.device("cuda", 0)
        ok = {}
        # --- query-row bands of one frame (C2 geometry, 6 iterations) ---
        spec = cvb.LookupSpec(4, 4)
        h, w = 135, 240
        sc = cvb.gen_scenario(0, (h, w, 256), 6, spec, coords_dtype=np.float32)
        bands = row_bands(h, world)
        a, b = bands[rank]
        for strict in (False, True):
            f1 = cvb.FeatureMap(torch.from_numpy(sc.f1[a:b].copy()).to(dev))
            f2 = cvb.FeatureMap(torch.from_numpy(sc.f2).to(dev))
            band = cvb.CorrSampler(f1, f2, spec, strict=strict)
            full = None
            if rank == 0:
                full = cvb.CorrSampler(cvb.FeatureMap(torch.from_numpy(sc.f1).to(dev)), f2, spec,
                                       strict=strict)
            same = True
            for c in sc.centroid_fields:
                got = band(torch.from_numpy(c[a:b].copy()).to(dev)).values
                gathered = gather_bands(got, bands)
                if rank == 0:
                    want = full(torch.from_numpy(c).to(dev)).values
                    same &= bool(torch.equal(gathered, want))
            ok[f"bands_strict={strict}"] = same
        # --- batch slices (C5-style, normalize) ---
        spec = cvb.LookupSpec(4, 4, True)
        batch = 3
        scs = [cvb.gen_scenario(s, (46, 62, 256), 4, spec, coords_dtype=np.float32)
               for s in range(batch)]
        slices = batch_slices(batch, world)
        s0, s1 = slices[rank]
        mine = scs[s0:s1]
        f1 = torch.stack([torch.from_numpy(s.f1) for s in mine]).to(dev)
        f2 = torch.stack([torch.from_numpy(s.f2) for s in mine]).to(dev)
        bs = cvb.BatchCorrSampler(f1, f2, spec)
        same = True
        for it in range(4):
            c = torch.stack([torch.from_numpy(s.centroid_fields[it]) for s in mine]).to(dev)
            gathered = gather_bands(bs(c), slices)
            if rank == 0:
                for p, s in enumerate(scs):
                    single = cvb.CorrSampler(torch.from_numpy(s.f1).to(dev),
                                             torch.from_numpy(s.f2).to(dev), spec)
                    for j in range(it + 1):
                        want = single(torch.from_numpy(s.centroid_fields[j]).to(dev)).values
                    same &= bool(torch.equal(gathered[p], want))
        ok["batch_slices"] = same
        dist.destroy_process_group()
        q.put((rank, ok))
    except Exception as exc:  # surface worker failures
        import traceback

        q.put((rank, traceback.format_exc()))


def test_two_ranks_share_the_gpu_and_reassemble_bitwise(cuda):
    world = 2
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=900) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    assert isinstance(results[0], dict), results[0]
    assert isinstance(results[1], dict), results[1]
    assert results[0] == {"bands_strict=False": True, "bands_strict=True": True,
                          "batch_slices": True}


def test_bench_two_rank_launch(cuda):
    """torchrun bench.py --gpus 2 (gloo, both ranks on the one GPU): one rank-0
    JSON line with the contract's keys, n_gpus 2, query-row bands."""
    env = dict(os.environ, CVB_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "bench.py"), "--gpus", "2", "--config", "C2", "--steps", "3",
           "--warmup", "3", "--no-e2e", "--no-compare", "--no-cpu-baseline"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-3000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["steps"] == 3 and line["warmup"] == 3
    assert line["config"]["parallelism"] == "query-row bands x2"
    assert line["value"] > 0 and line["ms_per_step"] > 0
    assert line["gpu_launches"] > 0
