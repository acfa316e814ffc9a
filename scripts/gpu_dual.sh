# dual-MMA race hunt: every candidate of l1.b1.c1 at N=256 and a few N for the first failing one
export CONV_Q_LIB=$PWD/paper_2202_06819_b200/libconvq_dual.so
python - <<'PY'
import subprocess, sys
sys.path.insert(0, ".")
import paper_2202_06819_b200 as cq
p = cq.ConvPlan(256, 56, 56, 256, 64, 1, 1, 1, 0, 8, relu=True)
for c in p.candidates():
    r = subprocess.run([sys.executable, "scripts/check_cfg.py", "l1.b1.c1", c, "256"], capture_output=True, text=True, timeout=None) if False else None
    try:
        r = subprocess.run([sys.executable, "scripts/check_cfg.py", "l1.b1.c1", c, "256"], capture_output=True, text=True, timeout=40)
        print(c, r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ("rc=%d " % r.returncode) + r.stderr.strip().splitlines()[-1][:100], flush=True)
    except subprocess.TimeoutExpired:
        print(c, "HANG (40 s)", flush=True)
PY
