"""bench.py's JSON-line contract (the driver parses it): the reference arm on CPU
(-m "not gpu"), the device arm on a B200 (-m gpu)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--workload", "resnet18_int8_b1", "--steps", "1", "--warmup", "0",
              "--ref-budget", "2"], timeout=300)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["unit"] == "images/s" and d["dtype"] == "int8" and d["config"]["workload"] == "resnet18_int8_b1"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_device_arm_contract():
    d = _run(["--steps", "5", "--warmup", "3", "--no-tune", "--no-cpu-baseline", "--no-k7", "--no-stem"],
             timeout=900)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"] == "resnet50_int8_b256" and d["dtype"] == "int8"
    r = d["roofline"]
    assert r["bound"] in ("tensor", "hbm") and 0 < r["frac"] <= 1 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 256 * 56 * 56 * 64 * 2 and e["d2h_bytes_per_step"] == 256 * 7 * 7 * 2048
    assert d["gpu_launches"] == 53 * 5
    assert d["clocks"]["sm_max_mhz"] > 0
