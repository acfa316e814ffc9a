"""Run one conv layer a few times (for ncu captures): python scripts/prof_layer.py
--workload resnet50 --layer l3.b1.c2 --batch 256 --bits 8 [--config NAME] [--reps 3]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2202_06819_b200 as cq  # noqa: E402
import workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="resnet50", choices=["resnet50", "resnet18", "table1"])
ap.add_argument("--layer", default="l3.b1.c2")
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--bits", type=int, default=8)
ap.add_argument("--config", default="")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
table = {"resnet50": [l for l, _ in wl.resnet50_layers()], "resnet18": [l for l, _ in wl.resnet18_layers()],
         "table1": wl.paper_table1_layers()}[a.workload]
g = wl.rng(9, 0)
if a.layer == "stem":   # ResNet conv1 through the s2d StemPlan
    L = "stem conv1 7x7/2 224x224x3->64 (s2d)"
    p = cq.StemPlan(a.batch, 224, 224, 3, 64, 7, 7, 3, a.bits, relu=True)
    xd = torch.from_numpy(wl.random_bytes(g, p.x_dims)).cuda()
    wd = torch.from_numpy(wl.random_bytes(g, p.w_dims)).cuda()
    sd = torch.cat([torch.full((64,), 0.01), torch.zeros(64)]).cuda()
    y = torch.empty((a.batch, 112, 112, 64 * a.bits // 8), dtype=torch.uint8, device="cuda")
else:
    L = {l.name: l for l in table}[a.layer]
    x, w, ss = wl.layer_inputs(g, L, a.batch, a.bits)
    p = cq.ConvPlan(a.batch, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, a.bits, relu=True)
    xd, wd, sd = (torch.from_numpy(t).cuda() for t in (x, w, ss))
    y = torch.empty((a.batch, L.P, L.Q, L.K * a.bits // 8), dtype=torch.uint8, device="cuda")
if a.config:
    p.set_config(p.candidates().index(a.config))
for _ in range(a.reps):
    p.run(xd, wd, sd, y)
torch.cuda.synchronize()
print(L, p.info().config)
