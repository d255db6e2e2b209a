"""bench.py's JSON line (the driver's contract): the reference arm on CPU, the GPU arm on a small
config. Checks the keys and their types, not performance."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def _common(d):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"):
        assert k in d, k
    assert d["metric"] == "line-region tests/s" and d["unit"] == "tests/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["vs_baseline"] is None
    assert "workload" in d["config"]
    assert d["scaling"] in ("weak", "strong")


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "2", "--steps", "1", "--warmup", "0"])
    _common(d)
    assert d["impl"] == "reference"
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["value"] == d["value"]
    assert c["cores"] >= 1 and c["os_cpu_count"] == os.cpu_count() and c["cpu_model"] and c["sample"]
    assert d["config"]["points_per_image"] == 17107
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run(["--config", "2", "--steps", "2", "--warmup", "3"])
    _common(d)
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["dtype"] in ("int32", "int64")
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("smem", "hbm") and 0 < r["frac"] and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"] and c["cpu_model"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
