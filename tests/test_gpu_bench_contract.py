"""bench.py keeps the driver's JSON-line contract (one line, the required keys,
a roofline with measured denominators, an end-to-end number with its copy
volumes, clocks, launch count) — run on the small C1 frame."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

from oracle import import_reference

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _run(*args, timeout=600):
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


def test_bench_line_contract(cuda):
    d = _run("--config", "C1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "e2e", "clocks", "gpu_launches"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["higher_is_better"] is False and d["value"] > 0
    assert "workload" in d["config"]
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert 0 < r["frac"] < 1 and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > d["value"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["clocks"]["sm_mhz"] > 0
    assert d["gpu_launches"] > 0


def test_reference_arm_line(cuda):
    if import_reference() is None:
        pytest.skip("oracle/_ref not built")
    d = _run("--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_bench_parity_against_the_reference(cuda):
    """The CPU-baseline leg's reference run checks the GPU's cost maps on the
    rows it times (every iteration): strict bitwise, fast within both gates."""
    if import_reference() is None:
        pytest.skip("oracle/_ref not built")
    d = _run("--config", "C1", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-compare",
             timeout=900)
    p = d["parity"]
    assert p["iterations"] == 12 and p["rows"][1] > p["rows"][0]
    assert p["strict_bitwise"] and p["pass"]
    assert p["fast_ref_gate"] <= 1e-5 and p["fast_ns_gate"] <= 1e-4
