"""NEXT-3: the B200 analog of the paper's ablation (section 4.4,
Figs. 15-16: accumulated and marginal speed-up of each optimisation per
ResNet-50 stage).

Every candidate of every ResNet-50 layer (batch 256, INT8, ReLU) is timed on
the device (conv_q_plan_time_candidates: back-to-back launches, median of 3
rounds), in the fused packed mode and in the unfused mode (s32 output +
conv_q_requant, the separate re-layout pass the fused epilogue replaces).
A design = a set of enabled features; its time for a layer = the fastest
candidate the features allow; a stage's time = the sum over its layers.

Features (each maps to candidate-name tokens):
  fused   requant + repack in the conv epilogue (else s32 out + conv_q_requant)
  halo    duplicate-aware A operand (_h; 3x3 s1 layers)
  pair    CTA pair, cta_group::2, M = 256 (_c2)                                     --
  ws      weight-stationary resident weights + MT2 units (_w, _m2)                 --
  split   split-K work units (_k<s>)
Accumulated: baseline (no feature), then + each feature in the order above.
Marginal: the full design with one feature removed.
INT4 vs INT8: the full design's time with INT4 operands at the same batch.

Writes a JSON (--out) and prints a markdown table.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_06819_b200 as cq  # noqa: E402
import workloads as wl  # noqa: E402

FEATURES = ["fused", "halo", "pair", "ws", "split"]


def feats_of(name: str) -> set:
    import re
    f = set()
    if "_h" in name:
        f.add("halo")
    if "_c2" in name:
        f.add("pair")
    if "_w" in name:
        f.add("ws")
    if re.search(r"_k\d", name):      # split-K suffix _k<s> (not the _kc<ch> field)
        f.add("split")
    return f


def time_requant(acc, ss, y, bits, reps=10):
    s = torch.cuda.current_stream()
    for _ in range(3):
        cq.requant(acc, ss, True, bits, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        e0.record(s)
        for _ in range(reps):
            cq.requant(acc, ss, True, bits, out=y)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    return sorted(ts)[1]


def layer_table(L, N, bits, g, reps):
    x, w, ss = wl.layer_inputs(g, L, N, bits)
    xd, wd, sd = (torch.from_numpy(a).cuda() for a in (x, w, ss))
    M = N * L.P * L.Q
    y = torch.empty((M, L.K * bits // 8), dtype=torch.uint8, device="cuda")
    y32 = torch.empty((M, L.K), dtype=torch.int32, device="cuda")
    plan = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
    names = plan.candidates()
    fused = plan.time_candidates(xd, wd, sd, y, warmup=2, reps=reps)
    plan.set_epilogue(True, cq.OUT_S32)
    s32 = plan.time_candidates(xd, wd, sd, y32, warmup=2, reps=reps)
    rq = time_requant(y32, sd, y, bits)
    del y32
    return {"names": names, "fused_us": fused, "s32_us": s32, "requant_us": rq}


def design_time(tab, feats: set) -> float:
    best = None
    for n, tf, ts in zip(tab["names"], tab["fused_us"], tab["s32_us"]):
        if not feats_of(n) <= feats:
            continue
        t = tf if "fused" in feats else (ts + tab["requant_us"] if ts > 0 else -1)
        if t > 0 and (best is None or t < best):
            best = t
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="profiles/r02_ablation.json")
    ap.add_argument("--from-raw", default="", help="recompute the tables from a saved _raw.json")
    args = ap.parse_args()
    if args.from_raw:
        raw = json.load(open(args.from_raw))
        tabs = {int(b): {tuple(int(v) for v in k.strip("()").split(",")): t for k, t in d.items()}
                for b, d in raw.items()}
        return report(args, tabs)
    cq.load()
    layers = [L for L, _ in wl.resnet50_layers()]
    uniq = {}
    for L in layers:
        uniq.setdefault((L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad), L)
    tabs = {8: {}, 4: {}}
    for bits in (8, 4):
        for k, L in uniq.items():
            g = wl.rng(7, hash(k) % 1000)
            tabs[bits][k] = layer_table(L, args.batch, bits, g, args.reps)
            print(f"[ablation] int{bits} {L.name} {k}: {len(tabs[bits][k]['names'])} candidates", file=sys.stderr)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out.replace(".json", "_raw.json"), "w") as f:   # raw per-candidate times first
        json.dump({str(b): {str(k): v for k, v in t.items()} for b, t in tabs.items()}, f)
    report(args, tabs)


def report(args, tabs):
    layers = [L for L, _ in wl.resnet50_layers()]
    uniq = {}
    for L in layers:
        uniq.setdefault((L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad), L)

    def stage_of(L):
        return L.name.split(".")[0]

    designs = {"baseline": set()}
    acc = set()
    for f in FEATURES:
        acc = acc | {f}
        designs["+" + f] = set(acc)
    full = set(FEATURES)
    for f in FEATURES:
        designs["full-" + f] = full - {f}
    stages = ["l1", "l2", "l3", "l4"]
    result = {"batch": args.batch, "features": FEATURES, "stages": {}, "per_shape": {}}
    for st in stages + ["all"]:
        ls = [L for L in layers if st == "all" or stage_of(L) == st]
        row = {}
        for dname, fs in designs.items():
            row[dname] = sum(design_time(tabs[8][(L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad)], fs) for L in ls)
        row["int4_full"] = sum(design_time(tabs[4][(L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad)], full)
                               for L in ls)
        result["stages"][st] = row
    for k, L in uniq.items():
        result["per_shape"][L.name] = {
            "shape": list(k), "int8": {d: design_time(tabs[8][k], fs) for d, fs in designs.items()},
            "int4_full": design_time(tabs[4][k], full),
            "requant_us_int8": tabs[8][k]["requant_us"],
            "candidates_int8": dict(zip(tabs[8][k]["names"], tabs[8][k]["fused_us"]))}
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(result, f, indent=1)
    # markdown: accumulated speed-up over the baseline, marginal = full / (full - f)
    print("| stage | baseline us | " + " | ".join("+" + f for f in FEATURES) + " | full us | "
          + " | ".join("marg " + f for f in FEATURES) + " | INT4/INT8 time |")
    print("|---" * (3 + 2 * len(FEATURES) + 1) + "|")
    for st in stages + ["all"]:
        r = result["stages"][st]
        b = r["baseline"]
        fullt = r["+" + FEATURES[-1]]
        acc_s = " | ".join(f"{b / r['+' + f]:.2f}x" for f in FEATURES)
        marg = " | ".join(f"{r['full-' + f] / fullt:.2f}x" for f in FEATURES)
        print(f"| {st} | {b:.1f} | {acc_s} | {fullt:.1f} | {marg} | {r['int4_full'] / fullt:.2f} |")


if __name__ == "__main__":
    main()
