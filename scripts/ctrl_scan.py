"""Bare-control-skeleton time (probe 7, instrumented build) vs batch: per-stage
slope and per-launch intercept.  python scripts/ctrl_scan.py layer config"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("CONV_Q_LIB", os.path.join(ROOT, "paper_2202_06819_b200", "libconvq_instr.so"))
sys.path.insert(0, ROOT)
import torch
import paper_2202_06819_b200 as cq, workloads as wl
name, cfg = sys.argv[1], sys.argv[2]
L = {l.name: l for l, _ in wl.resnet50_layers()}[name]
g = wl.rng(9, 0)
for N in (8, 32, 64, 128, 256):
    x, w, ss = wl.layer_inputs(g, L, N, 8)
    p = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, 8, relu=True)
    xd, wd, sd = (torch.from_numpy(t).cuda() for t in (x, w, ss))
    y = torch.empty((N, L.P, L.Q, L.K), dtype=torch.uint8, device="cuda")
    p.set_config(p.candidates().index(cfg))
    for _ in range(3): p.run(xd, wd, sd, y)
    res = []
    for reps in (1, 20):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps): p.run(xd, wd, sd, y)
        e1.record(); torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / reps * 1000)
    print(f"{name} {cfg} N={N:4d}: single {res[0]:7.1f} us  back-to-back {res[1]:7.1f} us", flush=True)
