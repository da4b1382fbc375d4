"""Multi-rank logic on CPU (gloo, world_size 2): row-band partition and the
band all-gather reassemble exactly the single-process result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_2505_16942_b200.parallel import batch_slices, gather_bands, row_bands


def test_row_bands_cover_and_align():
    for h in (1, 7, 8, 46, 135, 540):
        for world in (1, 2, 3, 4, 8):
            bands = row_bands(h, world)
            assert len(bands) == world
            assert bands[0][0] == 0 and bands[-1][1] == h
            for (a, b), (c, _) in zip(bands, bands[1:]):
                assert b == c
            for a, b in bands:
                assert a <= b and (a % 8 == 0 or a == b == h)
            sizes = [b - a for a, b in bands if b - a]
            assert max(sizes) - min(sizes) < 16  # one 8-row unit + the partial last unit


def test_batch_slices():
    assert batch_slices(64, 8) == [(8 * i, 8 * i + 8) for i in range(8)]
    s = batch_slices(10, 4)
    assert s[0] == (0, 3) and s[-1] == (8, 10)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, f1, f2, coords, want, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import corrvol_oracle as O

        bands = row_bands(f1.shape[0], world)
        a, b = bands[rank]
        local = O.lookup(f1, f2, coords, 2, 2, rows=slice(a, b))
        full = gather_bands(torch.from_numpy(local), bands)
        q.put((rank, bool(np.array_equal(full.numpy(), want))))
        dist.destroy_process_group()
    except Exception as exc:  # surface worker failures
        q.put((rank, repr(exc)))


@pytest.mark.parametrize("world", [2])
def test_band_gather_reassembles_full_output_gloo(world):
    from oracle import corrvol_oracle as O

    rng = np.random.default_rng(0)
    h, w, d = 21, 13, 8
    f1 = rng.standard_normal((h, w, d)).astype(np.float32)
    f2 = rng.standard_normal((h, w, d)).astype(np.float32)
    ys, xs = np.mgrid[0:h, 0:w]
    coords = np.stack([xs, ys], -1).astype(np.float64) + rng.uniform(-3, 3, (h, w, 2))
    want = O.lookup(f1, f2, coords, 2, 2)
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, f1, f2, coords, want, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert results == {r: True for r in range(world)}
