"""compute-sanitizer over every candidate family at cfg1 and edge sizes, the
residual epilogue with unsigned codes, and a two-layer chain with cross-launch
completion counters (-m gpu;
skipped when the tool is absent or the GPU pool's wrapper has closed it).  memcheck: out-of-bounds / misaligned
global and shared accesses; synccheck: invalid barrier use.  The async
pipeline (TMA, mbarriers, tcgen05) is the part a race or a wrong byte count
would break (round 1 hit a real pipeline race in the dual-MMA variant)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "synccheck"])
def test_compute_sanitizer(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, f"--tool={tool}", "--error-exitcode=17", "--print-limit=20", sys.executable,
           os.path.join(ROOT, "scripts", "sanitize_run.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses to run (earlier runs left GPUs
        # needing a reset); the last runs it allowed are recorded in DESIGN.md
        pytest.skip("compute-sanitizer closed on this GPU pool: " + out.strip().splitlines()[0][:200])
    assert r.returncode == 0, out[-4000:]
    assert "sanitize_run:" in out and "ERROR SUMMARY: 0 errors" in out, out[-4000:]
