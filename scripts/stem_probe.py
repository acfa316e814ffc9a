"""Measurement: ResNet conv1 (7x7/2 p3, 224x224x3 -> 64) at batch B as the s2d
StemPlan (every candidate timed) vs the direct ConvPlan on C padded to 32."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2202_06819_b200 as cq
import workloads as wl

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dev = torch.device("cuda", 0)
g = np.random.default_rng(1)
x = torch.from_numpy(wl.fp16_activations(g, B, 224, 224, 3)).to(dev)
wv = torch.from_numpy(wl.weight_values(g, 64, 7, 7, 3, bits)).to(dev)
ss = torch.cat([torch.full((64,), 0.01, device=dev), torch.zeros(64, device=dev)])
inv = 127 / 4 if bits == 8 else 7 / 3
y = torch.empty((B, 112, 112, 64 * bits // 8), dtype=torch.uint8, device=dev)
ops = 2 * B * 112 * 112 * 64 * 147


def timeit(fn, n=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


p = cq.StemPlan(B, 224, 224, 3, 64, 7, 7, 3, bits, relu=True)
xs = p.quantize(x, inv)
wp = p.pack_weights(wv)
print("s2d x_dims", p.x_dims, "w_dims", p.w_dims, "Kg", p.info().Kg)
print(f"s2d quantize: {timeit(lambda: p.quantize(x, inv, out=xs)):.1f} us  "
      f"({(x.numel() * 2 + xs.numel()) / 1e9:.3f} GB)")
for i, name in enumerate(p.candidates()):
    p.set_config(i)
    us = timeit(lambda: p.run(xs, wp, ss, y))
    print(f"  {name:32s} {us:8.1f} us  {ops / us / 1e6:8.1f} useful TOPS  "
          f"{(xs.numel() + y.numel()) / us / 1e3:7.1f} GB/s")
best = p.tune(xs, wp, ss, y, warmup=2, reps=5)
print("tuned:", p.info().config, p.info().tuned_us)
tot = timeit(lambda: (p.quantize(x, inv, out=xs), p.run(xs, wp, ss, y)))
print(f"stem total (s2d quantize + conv): {tot:.1f} us")
if "--direct" in sys.argv:
    Cp = cq.padded_channels(3, bits)
    xq = cq.quantize(x, inv, bits)
    wd = cq.pack_weights(torch.nn.functional.pad(wv, (0, Cp - 3)).contiguous(), bits)
    d = cq.ConvPlan(B, 224, 224, Cp, 64, 7, 7, 2, 3, bits, relu=True)
    d.tune(xq, wd, ss, y, warmup=1, reps=2)
    print("direct:", d.info().config, d.info().tuned_us, "us")
