"""Per-launch floor: a CUDA graph of 50 back-to-back launches (PDL) of a tiny conv
(one 128-row tile) for several configs, and of the tiny max-pool kernel.
python scripts/launch_floor.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2202_06819_b200 as cq, workloads as wl

def graph_time(fn, n=50):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(s); g.replay(); e1.record(s); torch.cuda.synchronize()
    torch.cuda.set_stream(torch.cuda.default_stream())
    return e0.elapsed_time(e1) * 1000 / n

gr = wl.rng(1, 1)
for (H, C, K, R) in [(8, 64, 64, 1), (8, 64, 64, 3), (16, 256, 256, 3)]:
    L = wl.Layer("t", H, H, C, K, R, R, 1, R // 2)
    x, w, ss = wl.layer_inputs(gr, L, 1, 8)
    xd, wd, sd = (torch.from_numpy(a).cuda() for a in (x, w, ss))
    y = torch.empty((L.P * L.Q, K), dtype=torch.uint8, device="cuda")
    p = cq.ConvPlan(1, H, H, C, K, R, R, 1, R // 2, 8, relu=True)
    for i, name in enumerate(p.candidates()):
        if __import__("re").search(r"_k\d", name):
            continue
        p.set_config(i)
        t = graph_time(lambda: p.run(xd, wd, sd, y))
        print(f"conv {H}x{H} {C}->{K} {R}x{R} {name:34s} {t:6.2f} us/launch", flush=True)
xp = torch.zeros((1, 16, 16, 64), dtype=torch.uint8, device="cuda")
print(f"maxpool 16x16x64: {graph_time(lambda: cq.maxpool(xp, 64, 3, 2, 1, 8)):6.2f} us/launch")
xq = torch.zeros((1, 16, 16, 64), dtype=torch.float16, device="cuda")
print(f"quantize 16x16x64: {graph_time(lambda: cq.quantize(xq, 1.0, 8)):6.2f} us/launch")
