"""Run every TileConfig candidate family once on small shapes (cfg1 and edge
sizes), packed and s32 outputs, for compute-sanitizer (memcheck / synccheck).
Used by tests/test_gpu_sanitizer.py; exits non-zero on any CUDA error."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_06819_b200 as cq  # noqa: E402
import workloads as wl  # noqa: E402

SHAPES = [(wl.CFG1, 1, 8), (wl.Layer("tail", 9, 11, 64, 64, 3, 3, 1, 1), 3, 8),
          (wl.Layer("1x1", 14, 14, 256, 256, 1, 1, 1, 0), 2, 8), (wl.Layer("s2", 13, 13, 128, 128, 3, 3, 2, 1), 2, 8),
          (wl.Layer("l4", 7, 7, 512, 512, 3, 3, 1, 1), 1, 8), (wl.CFG1, 1, 4),
          (wl.Layer("1x1", 14, 14, 256, 256, 1, 1, 1, 0), 2, 4)]
FAMILY = os.environ.get("SAN_FAMILY", "")     # optional substring filter on candidate names


def main():
    cq.load()
    g = np.random.default_rng(1)
    n = 0
    for L, N, bits in SHAPES:
        x, w, ss = wl.layer_inputs(g, L, N, bits)
        xd, wd, sd = (torch.from_numpy(a).cuda() for a in (x, w, ss))
        y = torch.empty((N * L.P * L.Q, L.K * bits // 8), dtype=torch.uint8, device="cuda")
        y32 = torch.empty((N * L.P * L.Q, L.K), dtype=torch.int32, device="cuda")
        plan = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits)
        for ci, name in enumerate(plan.candidates()):
            if FAMILY and FAMILY not in name:
                continue
            plan.set_config(ci)
            for relu, mode, out in ((True, cq.OUT_PACKED, y), (False, cq.OUT_PACKED, y), (False, cq.OUT_S32, y32)):
                plan.set_epilogue(relu, mode)
                plan.run(xd, wd, sd, out)
            torch.cuda.synchronize()
            n += 1
    xf = torch.randn(2, 30, 38, 3, device="cuda").half()
    sp = cq.StemPlan(2, 30, 38, 3, 64, 7, 7, 3, 8, relu=True)
    xs = sp.quantize(xf, 32.0)
    wp = sp.pack_weights(torch.randint(-128, 127, (64, 7, 7, 3), dtype=torch.int8, device="cuda"))
    ssd = torch.from_numpy(wl.scale_shift(g, 64, 147, 30, 70, 8)).cuda()
    ys = torch.empty((2, sp.P, sp.Q, 64), dtype=torch.uint8, device="cuda")
    for ci, _ in enumerate(sp.candidates()):
        sp.set_config(ci)
        sp.run(xs, wp, ssd, ys)
        n += 1
    cq.maxpool(ys, 64, 3, 2, 1, 8)
    cq.maxpool(ys, 64, 3, 2, 1, 8, uns=True)
    # residual epilogue (TMA skip slabs / register skips / split-K) with unsigned codes
    for L, N, bits in ((wl.Layer("res", 14, 14, 256, 256, 1, 1, 1, 0), 2, 8), (wl.Layer("res4", 9, 11, 64, 64, 3, 3, 1, 1), 2, 4)):
        x, w, ss = wl.layer_inputs(g, L, N, bits)
        xd, wd, sd = (torch.from_numpy(a).cuda() for a in (x, w, ss))
        sk = torch.from_numpy(wl.random_bytes(g, (N * L.P * L.Q, L.K * bits // 8))).cuda()
        y = torch.empty((N * L.P * L.Q, L.K * bits // 8), dtype=torch.uint8, device="cuda")
        plan = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
        plan.set_formats(True, True, True)
        plan.set_residual(sk, 0.5)
        for ci, name in enumerate(plan.candidates()):
            if FAMILY and FAMILY not in name:
                continue
            plan.set_config(ci)
            plan.run(xd, wd, sd, y)
            torch.cuda.synchronize()
            n += 1
    # two-layer chain with cross-launch completion counters (conv_q_plan_set_deps)
    L1, L2 = wl.Layer("d1", 14, 14, 128, 128, 3, 3, 1, 1), wl.Layer("d2", 14, 14, 128, 128, 1, 1, 1, 0)
    N = 2
    x, w1, s1 = wl.layer_inputs(g, L1, N, 8)
    _, w2, s2 = wl.layer_inputs(g, L2, N, 8)
    xd = torch.from_numpy(x).cuda()
    w1d, s1d, w2d, s2d = (torch.from_numpy(a).cuda() for a in (w1, s1, w2, s2))
    y1 = torch.empty((N, 14, 14, 128), dtype=torch.uint8, device="cuda")
    y2 = torch.empty((N, 14, 14, 128), dtype=torch.uint8, device="cuda")
    f1 = torch.zeros(1, dtype=torch.int32, device="cuda")
    f2 = torch.zeros(1, dtype=torch.int32, device="cuda")
    p1 = cq.ConvPlan(N, 14, 14, 128, 128, 3, 3, 1, 1, 8, relu=True)
    p2 = cq.ConvPlan(N, 14, 14, 128, 128, 1, 1, 1, 0, 8, relu=True)
    p1.set_deps(None, None, f1)
    p2.set_deps(f1, None, f2)
    for c1 in range(0, len(p1.candidates()), 3):
        p1.set_config(c1)
        for c2 in range(0, len(p2.candidates()), 5):
            p2.set_config(c2)
            f1.zero_()
            f2.zero_()
            p1.run(xd, w1d, s1d, y1)
            p2.run(y1, w2d, s2d, y2)
            torch.cuda.synchronize()
            n += 1
    torch.cuda.synchronize()
    print(f"sanitize_run: {n} candidate configs ran")


if __name__ == "__main__":
    main()
