"""bench.py's JSON-line contract on the CPU: the reference arm (the oracle on the host cores,
DESIGN.md §8) prints one line with the keys the driver reads, with its cpu_baseline and e2e
objects; bench.py parses its options without a GPU.  The GPU arm's line is checked on the
B200 (the round-end bench run) -- its keys are listed in DESIGN.md §8."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "gray_scott_cell_updates_per_s"
    assert d["unit"] == "cell-updates/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["steps"] == 1 and d["warmup"] == 1 and d["n_gpus"] == 1
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"] == "gray_scott_dopri5_adaptive_512^3_per_gpu"


import pytest  # noqa: E402


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """The GPU arm on a small grid: one JSON line with roofline, clocks, gpu_launches, e2e and
    cpu_baseline objects."""
    r = subprocess.run([sys.executable, "bench.py", "--n", "64", "--legs", "adaptive,rk4,e2e,cpu", "--steps", "3",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks", "e2e",
              "cpu_baseline"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["dtype"] == "f64" and d["gpu_launches"] > 0
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["achieved"] > 0 and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 64 ** 3 * 2 * 8
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert "rk4" in d["extra"] and d["extra"]["rk4"]["value"] > 0
    assert rf["rk4_512"]["value"] > 0 and rf["rk4_512"]["frac"] > 0
    assert d["config"]["accepted_per_step"] > 0
