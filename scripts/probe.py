"""Time layers in normal / loads-only / MMA-only probe modes for every candidate.
python scripts/probe.py l3.b1.c2 l1.b0.c2 ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# probe modes exist only in the measurement build (CONVQ_INSTRUMENT=1 python paper_2202_06819_b200/_build.py)
os.environ.setdefault("CONV_Q_LIB", os.path.join(ROOT, "paper_2202_06819_b200", "libconvq_instr.so"))
CODE = r'''
import os, sys, json
sys.path.insert(0, %r)
import torch, numpy as np
import paper_2202_06819_b200 as cq, workloads as wl
name, N, bits = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
g = wl.rng(9, 0)
if name == "stem":
    p = cq.StemPlan(N, 224, 224, 3, 64, 7, 7, 3, bits, relu=True)
    xd = torch.from_numpy(wl.random_bytes(g, p.x_dims)).cuda()
    wd = torch.from_numpy(wl.random_bytes(g, p.w_dims)).cuda()
    sd = torch.cat([torch.full((64,), 0.01), torch.zeros(64)]).cuda()
    y = torch.empty((N, 112, 112, 64 * bits // 8), dtype=torch.uint8, device="cuda")
else:
    L = {l.name: l for l, _ in getattr(wl, os.environ.get("PROBE_NET", "resnet50") + "_layers")()}[name]
    x, w, ss = wl.layer_inputs(g, L, N, bits)
    p = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
    xd, wd, sd = (torch.from_numpy(t).cuda() for t in (x, w, ss))
    y = torch.empty((N, L.P, L.Q, L.K * bits // 8), dtype=torch.uint8, device="cuda")
res = {}
flt = os.environ.get("PROBE_CFG", "")
for i, cname in enumerate(p.candidates()):
    if flt and cname not in flt.split(","):
        continue
    p.set_config(i)
    for _ in range(3): p.run(xd, wd, sd, y)
    torch.cuda.synchronize()
    # 20 launches captured as one CUDA graph: device time, not the binding's ~13 us per call
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(20): p.run(xd, wd, sd, y)
    gr.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    gr.replay()
    e1.record(); torch.cuda.synchronize()
    res[cname] = round(e0.elapsed_time(e1) / 20 * 1000, 1)
print(json.dumps(res))
''' % ROOT
for name in sys.argv[1:]:
    out = {}
    MODES = [int(m) for m in os.environ.get('PROBE_MODES', '0,1,2,3,4,7').split(',')]
    for mode in MODES:
        env = dict(os.environ, CONV_Q_PROBE=str(mode))
        r = subprocess.run([sys.executable, "-c", CODE, name, os.environ.get("PROBE_N", "256"),
                            os.environ.get("PROBE_BITS", "8")], env=env, capture_output=True, text=True)
        out[mode] = r.stdout.strip() or r.stderr[-400:]
    print(name)
    import json
    d = {m: json.loads(v) if v.startswith("{") else v for m, v in out.items()}
    if all(isinstance(v, dict) for v in d.values()) and len(d) < 6:
        for c in d[MODES[0]]:
            print(f"  {c:26s} " + "  ".join(f"probe{m} {d[m][c]:7.1f}" for m in MODES) + " us")
    elif all(isinstance(v, dict) for v in d.values()):
        for c in d[0]:
            print(f"  {c:26s} normal {d[0][c]:7.1f}  noMMA {d[1][c]:7.1f}  noLoad {d[2][c]:7.1f}  "
                  f"ctrl+epi {d[3][c]:7.1f}  noEpi {d[4][c]:7.1f}  ctrl-only {d[7][c]:7.1f} us")
    else:
        print(d)
