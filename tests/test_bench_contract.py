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
    d = _run(["--steps", "5", "--warmup", "3", "--no-tune", "--no-cpu-baseline", "--no-k7"], timeout=900)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"] == "resnet50_int8_b256" and d["dtype"] == "int8"
    r = d["roofline"]
    assert r["bound"] in ("tensor", "hbm") and 0 < r["frac"] <= 1 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 256 * 224 * 224 * 3 * 2 and e["d2h_bytes_per_step"] == 256 * 7 * 7 * 2048
    assert d["gpu_launches"] == 55 * 5          # s2d quantize, conv1, max pool, 52 convs
    assert d["config"]["conv_layers_per_step"] == 53
    assert d["clocks"]["sm_max_mhz"] > 0
    assert d["parity_ok"] is True and d["parity"]["launches_checked"] == 54


@pytest.mark.gpu
def test_device_arm_two_ranks_one_gpu_gloo():
    """The N > 1 path end to end (strong scaling: the global batch split across
    two ranks, weight broadcast, max-over-ranks timing, parity on each shard)
    with two processes sharing the one GPU over gloo."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", "resnet18_int8_b1", "--batch", "4",
           "--dist-backend", "gloo", "--no-tune", "--no-k7", "--no-cpu-baseline", "--gather"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["global_batch"] == 4 and d["config"]["per_gpu_batch"] == 2
    assert d["parity_ok"] is True
    assert d["gather"]["bytes_total"] == 4 * 7 * 7 * 512
