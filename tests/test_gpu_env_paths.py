"""Opt-in launch paths read once per process from the environment, each run
in a fresh interpreter and compared with the default path of this process:
  * CVB_PDL=1 — programmatic dependent launch on every per-iteration edge
    (csrc/common.cu; the default uses it within an iteration only) and
    CVB_PDL=0 — plain stream-ordered launches: outputs bit-identical;
  * CVB_TC_DEBUG=16 — the contraction's role timeline (debug only): same
    outputs, and the dump file is written.
"""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2505_16942_b200 as cvb

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
DIMS, N_ITER, SEED = (45, 70, 64), 4, 11

SCRIPT = r"""
import sys, numpy as np, torch
import paper_2505_16942_b200 as cvb
spec = cvb.LookupSpec(4, 3)
sc = cvb.gen_scenario({seed}, {dims}, {n}, spec, coords_dtype=np.float32)
dev = torch.device("cuda:0")
s = cvb.CorrSampler(cvb.FeatureMap(torch.from_numpy(sc.f1).to(dev)),
                    cvb.FeatureMap(torch.from_numpy(sc.f2).to(dev)), spec)
outs = [s(cvb.CentroidField(torch.from_numpy(c).to(dev))).values.cpu().numpy()
        for c in sc.centroid_fields]
np.save(sys.argv[1], np.stack(outs))
"""


def _default_outputs(cuda):
    spec = cvb.LookupSpec(4, 3)
    sc = cvb.gen_scenario(SEED, DIMS, N_ITER, spec, coords_dtype=np.float32)
    s = cvb.CorrSampler(cvb.FeatureMap(torch.from_numpy(sc.f1).to(cuda)),
                        cvb.FeatureMap(torch.from_numpy(sc.f2).to(cuda)), spec)
    return np.stack([s(cvb.CentroidField(torch.from_numpy(c).to(cuda))).values.cpu().numpy()
                     for c in sc.centroid_fields])


def _run(tmp_path, env_extra):
    out = tmp_path / "out.npy"
    env = dict(os.environ, **env_extra)
    env["PYTHONPATH"] = str(ROOT) + os.pathsep + env.get("PYTHONPATH", "")
    code = SCRIPT.format(seed=SEED, dims=DIMS, n=N_ITER)
    res = subprocess.run([sys.executable, "-c", code, str(out)], env=env, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    return np.load(out)


def test_pdl_launches_bit_identical(cuda, tmp_path):
    want = _default_outputs(cuda)
    got = _run(tmp_path, {"CVB_PDL": "1"})
    assert np.array_equal(got, want)
    got = _run(tmp_path, {"CVB_PDL": "0"})
    assert np.array_equal(got, want)


def test_contraction_timeline_debug_path(cuda, tmp_path):
    want = _default_outputs(cuda)
    ts = tmp_path / "ts.bin"
    got = _run(tmp_path, {"CVB_TC_DEBUG": "16", "CVB_TC_TS_FILE": str(ts)})
    assert np.array_equal(got, want)
    assert ts.exists() and ts.stat().st_size == N_ITER * 4 * 64 * 32 * 8
