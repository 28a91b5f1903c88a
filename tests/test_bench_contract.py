"""bench.py's JSON line: the keys the driver and the judge read (reference arm on the CPU,
our arm on the GPU at the small config 1)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
             "gpu_launches", "cpu_baseline"}


def test_reference_arm_line_cpu():
    d = run_bench("--impl", "reference", "--config", "cfg1", "--steps", "1", "--warmup", "1")
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["metric"] == "frames/s" and d["unit"] == "frames/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["gpu_launches"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "frames/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("cfg1")


@pytest.mark.gpu
def test_our_arm_line_gpu():
    d = run_bench("--config", "cfg1", "--steps", "20", "--warmup", "3", "--cpu-seconds", "1")
    assert BASE_KEYS <= set(d) and {"roofline", "clocks", "kernels"} <= set(d)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3
    assert d["gpu_launches"] > 0 and d["dtype"] == "f32"
    roof = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(roof)
    assert 0 < roof["frac"] < 1 and roof["peak"] > 0
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["value"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    B = d["arm"]["batch"]  # frames per launch: every timed frame solve ran 10 iterations
    assert d["solves_checked"] == 20 * B and e2e["solves_checked"] == 20 * B
    ref = run_bench("--impl", "reference", "--config", "cfg1", "--steps", "1", "--warmup", "1")
    assert ref["config"] == d["config"]  # the two arms describe the same workload
