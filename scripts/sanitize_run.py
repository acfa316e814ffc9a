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
    torch.cuda.synchronize()
    print(f"sanitize_run: {n} candidate configs ran")


if __name__ == "__main__":
    main()
