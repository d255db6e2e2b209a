"""The committed bench lines under profiles/ are recomputable from themselves (VERDICT r1, item 2:
"roofline recomputable from the line alone"): value = tests per step / time per step, roofline.frac
= achieved / peak, achieved = algorithmic bytes per launch / the kernel's average launch time, the
kernel's share = its launches' time / the step time, and the ncu DRAM byte count attached to the
default line belongs to the profiled build and is not below the launch's algorithmic bytes."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")


def _line(name):
    with open(os.path.join(P, name)) as f:
        return json.loads(f.readline())


@pytest.mark.parametrize("name", ["r02_bench_default.jsonl", "r02_bench_c5_int64.jsonl", "r02_bench_c3.jsonl", "r02_bench_c4.jsonl"])
def test_bench_line_recomputable(name):
    d = _line(name)
    assert d["metric"] == "line-region tests/s" and d["n_gpus"] == 1
    assert d["value"] == pytest.approx(d["tests_per_step"] / (d["ms_per_step"] * 1e-3), rel=1e-6)
    r = d["roofline"]
    assert r["bound"] == "smem" and r["unit"] == "TB/s"
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-9)
    assert r["achieved"] == pytest.approx(r["algorithmic_bytes_per_launch"] / (r["avg_launch_ms"] * 1e-3) / 1e12, rel=1e-6)
    assert r["algorithmic_bytes_per_launch"] == pytest.approx(8 * r["raster_steps_per_launch"], rel=1e-9)
    share = r["avg_launch_ms"] * r["launches"] / (d["ms_per_step"] * d["steps"])
    assert r["kernel_share_of_step"] == pytest.approx(share, rel=1e-2)   # per-call device times vs the whole timed region
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["ms_per_step"] > d["ms_per_step"]
    assert e["value"] == pytest.approx(d["tests_per_step"] / (e["ms_per_step"] * 1e-3), rel=1e-6)
    assert d["gpu_launches"] > 0 and d["clocks"]["reasons"] == []


def test_default_line_carries_same_build_traffic():
    d = _line("r02_bench_default.jsonl")
    t = json.load(open(os.path.join(P, "ncu_traffic.json")))
    r = d["roofline"]
    assert d["dtype"] == "int32" and d["config"]["points_per_image"] == 16000000
    assert r["traffic"] is not None and "same build" in r["ncu"]
    h = r["hbm"]
    assert h["traffic"] == r["traffic"] and h["traffic"] >= h["traffic_launch_algorithmic_bytes"]
    assert h["traffic"] / h["traffic_launch_algorithmic_bytes"] < 1.1    # no wasted re-reads
    assert t["libhht_build_id"] in open(os.path.join(P, "r02_summary.md")).read()
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] == c["os_cpu_count"]
