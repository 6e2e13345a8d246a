"""bench.py's N = 1 line carries every key of the driver's contract (GPU).

The driver parses the last stdout line of `python bench.py --gpus N --steps K
--warmup W`; a small run here checks the keys and their consistency (value =
rows·features / time, the roofline fraction, the library-counted e2e bytes,
the timed region's clocks) — not the numbers, which bench.py measures at the
BASELINE size.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    cmd = [sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "1", "--steps", "5", "--warmup", "3",
           "--no-variants", "--rows", "400000", "--trees", "1"]
    r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "gpu_launches", "clocks"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["steps"] == 5 and line["warmup"] == 3
    cfg = line["config"]
    assert cfg["workload"].startswith("higgs-400000x28-k64") and cfg["rows_total"] == 400000
    rows_features = cfg["rows_total"] * cfg["features"]
    assert abs(line["value"] - rows_features / (line["ms_per_step"] / 1e3)) <= 1e-6 * line["value"]
    roof = line["roofline"]
    assert roof["unit"] == "GB/s" and roof["peak"] > 0
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    e2e = line["e2e"]
    for key in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step", "ms_per_step"):
        assert key in e2e, key
    # the root (contiguous ids: none uploaded) at 8-16 B per row of g/h, the bins back
    assert 8 * 400_000 <= e2e["h2d_bytes_per_step"] <= 16 * 400_000
    assert e2e["d2h_bytes_per_step"] == 28 * 64 * 24  # hbg_bin = {double, double, int64}
    assert line["gpu_launches"] >= line["steps"]
    cpu = line["cpu_baseline"]
    assert cpu["kind"] in ("reference", "port") and cpu["cores"] >= 1 and cpu["value"] > 0
    assert "sm_mhz" in line["clocks"] and "reasons" in line["clocks"]


def test_reference_arm_line_matches_our_arm():
    """`bench.py --impl reference`: the reference's own CPU path on the same
    workload — the same metric, unit and config as our arm's line."""
    ours = [sys.executable, os.path.join(REPO, "bench.py"), "--steps", "3", "--warmup", "3", "--no-variants",
            "--no-cpu-baseline", "--rows", "300000", "--trees", "1"]
    ref = [sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "2", "--warmup", "1",
           "--rows", "300000"]
    lines = []
    for cmd in (ours, ref):
        r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        lines.append(json.loads(r.stdout.strip().splitlines()[-1]))
    a, b = lines
    assert b["impl"] == "reference"
    for key in ("metric", "unit", "higher_is_better", "n_gpus", "scaling", "config"):
        assert a[key] == b[key], key
    assert b["value"] > 0 and b["cpu_baseline"]["kind"] in ("reference", "port")
    assert b["e2e"]["value"] == b["value"] and b["e2e"]["h2d_bytes_per_step"] == 0
