import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2202_06819_b200 as cq, workloads as wl, oracle
name, cfg, N = sys.argv[1], sys.argv[2], int(sys.argv[3])
L = {l.name: l for l, _ in wl.resnet50_layers()}[name]
g = wl.rng(9, 0)
x, w, ss = wl.layer_inputs(g, L, N, 8)
p = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, 8, relu=True)
p.set_config(p.candidates().index(cfg))
xd, wd, sd = (torch.from_numpy(t).cuda() for t in (x, w, ss))
y = torch.full((N, L.P, L.Q, L.K), 0xA5, dtype=torch.uint8, device="cuda")
p.run(xd, wd, sd, y); torch.cuda.synchronize()
M = N * L.P * L.Q
pix = np.unique(np.concatenate([np.arange(0, min(M, 300)), g.integers(0, M, 300)])).astype(np.int64)
ref = oracle.conv_q(x, w, L.C, L.stride, L.pad, 8, ss, True, pix=pix)
got = y.cpu().numpy().reshape(M, -1)[pix]
bad = np.argwhere((got != ref).any(1))
print(name, cfg, N, "OK" if bad.size == 0 else f"MISMATCH rows {pix[bad[:5,0]]} of {len(bad)}")
