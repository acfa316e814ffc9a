"""Per-candidate launch times of a layer with and without the fused residual
add (and with unsigned codes): python scripts/res_cands.py l1.b0.c3 [batch]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_06819_b200 as cq  # noqa: E402
import workloads as wl  # noqa: E402

name = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 256
L = dict((l.name, l) for l, _ in wl.resnet50_layers())[name]
g = wl.rng(3, 3)
x, w, ss = wl.layer_inputs(g, L, N, 8)
xd, wd, sd = (torch.from_numpy(a).cuda() for a in (x, w, ss))
y = torch.empty((N * L.P * L.Q, L.K), dtype=torch.uint8, device="cuda")
sk = torch.from_numpy(wl.random_bytes(g, (N * L.P * L.Q, L.K))).cuda()
rows = {}
for mode in ("plain", "res", "uns", "res_uns"):
    p = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, 8, relu=True,
                    x_uns="uns" in mode, y_uns="uns" in mode)
    if "res" in mode:
        if "uns" in mode:
            p.set_formats(True, True, True)
        p.set_residual(sk, 0.5)
    for n, t in zip(p.candidates(), p.time_candidates(xd, wd, sd, y, warmup=2, reps=10)):
        rows.setdefault(n, {})[mode] = t
print(f"{name} N={N}")
print("%-36s %9s %9s %9s %9s" % ("config", "plain", "res", "uns", "res_uns"))
for n, r in sorted(rows.items(), key=lambda kv: kv[1].get("plain", 1e9)):
    print("%-36s %9.1f %9.1f %9.1f %9.1f" % (n, r.get("plain", -1), r.get("res", -1), r.get("uns", -1), r.get("res_uns", -1)))
