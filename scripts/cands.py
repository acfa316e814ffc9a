"""Time every TileConfig candidate of a layer (CUDA events, back-to-back launches):
python scripts/cands.py <layer> [batch] [bits]   (TRACE_NET=resnet50|resnet18)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2202_06819_b200 as cq, workloads as wl
name = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 256
bits = int(sys.argv[3]) if len(sys.argv) > 3 else 8
net = os.environ.get("TRACE_NET", "resnet50")
L = {l.name: l for l, _ in getattr(wl, net + "_layers")()}[name]
g = wl.rng(9, 0)
x, w, ss = wl.layer_inputs(g, L, N, bits)
p = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
xd, wd, sd = (torch.from_numpy(t).cuda() for t in (x, w, ss))
y = torch.empty((N, L.P, L.Q, L.K * bits // 8), dtype=torch.uint8, device="cuda")
res = []
for i, cname in enumerate(p.candidates()):
    p.set_config(i)
    for _ in range(3): p.run(xd, wd, sd, y)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20): p.run(xd, wd, sd, y)
    e1.record(); torch.cuda.synchronize()
    res.append((e0.elapsed_time(e1) / 20 * 1000, cname))
ops = 2 * N * L.P * L.Q * L.K * L.C * L.R * L.S
for us, cname in sorted(res):
    print(f"{name} {cname:30s} {us:8.1f} us  {ops / us / 1e6:7.1f} TOPS")
