"""Config 5 of BASELINE.json: per-layer shape sweep, INT8 and INT4, every tile-config
candidate timed on the device -- the B200 analog of the paper's Table 1
(Baseline / Exhaustive / Searched time per ResNet-50 stage,
"Speed-up" row).  Here "default" is the plan's pre-tuning pick, "best" the
exhaustive minimum over the candidate set (what conv_q_plan_tune selects),
"worst" the slowest candidate; speed-up = default / best.

Also checks config invariance on every shape: all candidates must produce
byte-identical output (integer accumulation; DESIGN reading 10).

Shape sets:
  S1  PAPER.md Table 1 shapes at N = 8 (3x3 s1 p1, K = C)
  S2  the 23 unique ResNet-50 conv shapes at N = 32
  S3  C = K in {64..2048} x {1x1, 3x3} x {s1 at 28x28, s2 at 56x56}, N = 32

python scripts/sweep.py [--sets S1,S2,S3] [--bits 8,4] [--reps 10] [--out profiles/r01_sweep.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2202_06819_b200 as cq  # noqa: E402
import workloads as wl  # noqa: E402


def shape_sets(names):
    out = []
    if "S1" in names:
        out += [("S1", L, 8) for L in wl.paper_table1_layers()]
    if "S2" in names:
        seen = set()
        for L, _ in wl.resnet50_layers():
            key = (L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad)
            if key not in seen:
                seen.add(key)
                out.append(("S2", L, 32))
    if "S3" in names:
        for c in (64, 128, 256, 512, 1024, 2048):
            for r in (1, 3):
                for st, hw in ((1, 28), (2, 56)):
                    out.append(("S3", wl.Layer(f"c{c}_{r}x{r}_s{st}", hw, hw, c, c, r, r, st, (r - 1) // 2), 32))
    return out


def time_config(p, xd, wd, sd, y, reps):
    """Device time per launch: `reps` back-to-back launches captured in one CUDA
    graph (as in a layer sequence: no host launch overhead, PDL overlap kept),
    replayed 3 times, median."""
    p.run(xd, wd, sd, y)   # split-K workspace / tensor maps set up outside capture
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                p.run(xd, wd, sd, y, stream=s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps * 1000.0)
    return sorted(ts)[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sets", default="S1,S2,S3")
    ap.add_argument("--bits", default="8,4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    rows = []
    t_start = time.time()
    for bits in [int(b) for b in a.bits.split(",")]:
        for si, (set_name, L, N) in enumerate(shape_sets(a.sets.split(","))):
            g = wl.rng(5, si)
            x, w, ss = wl.layer_inputs(g, L, N, bits)
            xd, wd, sd = (torch.from_numpy(t).cuda() for t in (x, w, ss))
            y = torch.empty((N, L.P, L.Q, L.K * bits // 8), dtype=torch.uint8, device="cuda")
            p = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
            default = p.info().config_index
            names = p.candidates()
            ref = None
            invariant = True
            times = []
            for i, nm in enumerate(names):
                p.set_config(i)
                us = time_config(p, xd, wd, sd, y, a.reps)
                out = y.clone()
                if ref is None:
                    ref = out
                elif not torch.equal(ref, out):
                    invariant = False
                times.append((us, nm))
            ops = 2 * L.macs(N)
            best = min(times)
            worst = max(times)
            dflt = times[default]
            row = {"set": set_name, "layer": L.name, "N": N, "H": L.H, "W": L.W, "C": L.C, "K": L.K, "R": L.R,
                   "stride": L.stride, "pad": L.pad, "bits": bits, "candidates": len(names),
                   "best_us": round(best[0], 2), "best_config": best[1], "best_tops": round(ops / best[0] / 1e6, 1),
                   "default_us": round(dflt[0], 2), "default_config": dflt[1],
                   "worst_us": round(worst[0], 2), "worst_config": worst[1],
                   "speedup_best_vs_default": round(dflt[0] / best[0], 3),
                   "speedup_best_vs_worst": round(worst[0] / best[0], 3),
                   "config_invariant_bytes": invariant}
            rows.append(row)
            print(f"{set_name} b{bits} {L.name:14s} N={N:3d} {L.H}x{L.W} {L.C}->{L.K} {L.R}x{L.S} s{L.stride}: "
                  f"best {best[0]:8.1f}us {row['best_tops']:7.1f} TOPS ({best[1]}), default {dflt[0]:8.1f}us, "
                  f"worst {worst[0]:8.1f}us, x{row['speedup_best_vs_default']:.2f} vs default, "
                  f"{len(names)} cands, invariant={invariant}", flush=True)
            del p, xd, wd, sd, y, ref
    print(f"# {len(rows)} shapes in {time.time() - t_start:.0f} s; all config-invariant: "
          f"{all(r['config_invariant_bytes'] for r in rows)}")
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"device": torch.cuda.get_device_name(0), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
