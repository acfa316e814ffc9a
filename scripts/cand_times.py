"""Graph-timed per-candidate times of ResNet layers at a batch:
python scripts/cand_times.py [batch] layer ...   (CT_BITS=4|8, CT_NET=resnet50|resnet18, CT_TOP=10)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2202_06819_b200 as cq, workloads as wl
N = int(sys.argv[1])
bits = int(os.environ.get("CT_BITS", "8"))
net = os.environ.get("CT_NET", "resnet50")
top = int(os.environ.get("CT_TOP", "10"))
layers = dict((l.name, l) for l, _ in getattr(wl, net + "_layers")())
for name in sys.argv[2:]:
    L = layers[name]
    g = wl.rng(3, 3)
    x, w, ss = wl.layer_inputs(g, L, N, bits)
    xd, wd, sd = (torch.from_numpy(a).cuda() for a in (x, w, ss))
    y = torch.empty((N * L.P * L.Q, L.K * bits // 8), dtype=torch.uint8, device="cuda")
    p = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
    ts = p.time_candidates(xd, wd, sd, y, warmup=2, reps=20)
    print(f"{name} N={N} bits={bits}")
    for n, t in sorted(zip(p.candidates(), ts), key=lambda kv: kv[1] if kv[1] > 0 else 1e9)[:top]:
        print(f"   {n:36s} {t:7.2f} us")
