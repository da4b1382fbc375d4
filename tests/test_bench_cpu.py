"""bench.py's CPU-side contract (no GPU): the reference arm's JSON line at C1
(the reference's own CPU-runnable case) and the helpers both arms share."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def test_workload_string_is_shared_and_host_info():
    import bench

    assert bench.workload("C4") == ("C4 540x960 features D=256 L=4 r=4 12 iterations, "
                                    "one image pair per step")
    assert "normalize" in bench.workload("C3")
    assert bench.workload("C5", 8).startswith("C5 270x480") and "batch of 8" in bench.workload(
        "C5", 8)
    info = bench.host_info()
    assert info["nproc"] >= 1 and info["affinity_cores"] >= 1


def test_reference_arm_line_c1(reference):
    if reference is None:
        pytest.skip("oracle/_ref (the reference package) is not built")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--config", "C1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    import bench

    assert line["impl"] == "reference" and line["unit"] == "ms/iter"
    assert line["higher_is_better"] is False
    assert line["config"]["workload"] == bench.workload("C1")
    # 46 rows = six 8-row bands: covered by the workers when the host has 6 cores
    ext = line["extrapolation"]
    assert ext["frame_rows"] == 46 and 1.0 <= ext["factor"] <= 46 / 8
    assert line["ms_per_step"] > 0 and line["value"] > 0
    assert line["e2e"] == {"value": line["value"], "unit": "ms/iter", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
