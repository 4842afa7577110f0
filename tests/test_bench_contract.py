"""bench.py's JSON-line contract, run as the driver runs it: the reference
arm (the CPU oracle) here on the CPU, our arm on the GPU (-m gpu) at a small
config.  Checks the keys and their types, not the numbers."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def run(args, timeout):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                       timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1"], 600)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["metric"] == "grover_amp_updates_per_s" and d["value"] > 0 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("c1")


@pytest.mark.gpu
def test_our_arm_line():
    d = run(["--config", "c3", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"], 900)
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["higher_is_better"] is True and d["scaling"] in ("weak", "strong") and d["data"] == "synthetic"
    assert d["config"]["workload"].startswith("c3") and "l2" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and 0 < r["frac"] <= 1.5 and r["achieved"] == pytest.approx(
        r["frac"] * r["peak"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["check"]["abs_err"] < 1e-6  # the timed run's marked mass vs the closed form
