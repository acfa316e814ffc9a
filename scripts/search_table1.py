"""NEXT-4 evidence: the B200 analog of PAPER.md Table 1 and
of the diversity-aware search comparison (Fig. 14).

For each 3x3 s1 p1 convolution of ResNet-50 stages 2-5 at N = 8 (the paper's
shapes, 1,849,688,064 ops each) and for extra ResNet-50 b256 layers given on
the command line:
  baseline    the plan's untuned default TileConfig (the analog of the paper's
              "TVM main branch" baseline)
  exhaustive  every TileConfig candidate timed (conv_q_plan_time_candidates,
              default runtime knobs) -- the current a7 tuner
  searched    conv_q_plan_search over the enlarged space (TileConfig x split-K x
              epilogue wait x L2 policy x rotation x grid), `trials`
              measurements, diversity-aware selection on
  autotvm     the same search with diversity off (one mutant per chain)
plus each search's best-so-far curve by trial.  All times: graph-timed device
microseconds per launch (the tuner's own timing loop).

python scripts/search_table1.py OUT.json [trials] [bits] [layer@N ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2202_06819_b200 as cq
import workloads as wl

out = sys.argv[1]
trials = int(sys.argv[2]) if len(sys.argv) > 2 else 128
bits_list = [int(b) for b in sys.argv[3].split(",")] if len(sys.argv) > 3 else [8, 4]
extra = sys.argv[4:]
r50 = dict((l.name, l) for l, _ in wl.resnet50_layers())
jobs = [(L, 8, f"table1.{L.name}") for L in wl.paper_table1_layers()]
for e in extra:
    name, n = e.split("@")
    jobs.append((r50[name], int(n), f"resnet50.{name}@{n}"))

rows = []
for bits in bits_list:
    for L, N, tag in jobs:
        g = wl.rng(9, 9)
        x, w, ss = wl.layer_inputs(g, L, N, bits)
        xd, wd, sd = (torch.from_numpy(a).cuda() for a in (x, w, ss))
        y = torch.empty((N * L.P * L.Q, L.K * bits // 8), dtype=torch.uint8, device="cuda")
        row = {"layer": tag, "bits": bits, "N": N, "shape": f"{L.H}x{L.W} {L.C}->{L.K} {L.R}x{L.S} s{L.stride}",
               "ops": 2 * N * L.P * L.Q * L.K * L.C * L.R * L.S}
        p = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
        names = p.candidates()
        sizes, nvalid = p.space()
        row["candidates"] = len(names)
        row["space_points"] = nvalid
        ts = p.time_candidates(xd, wd, sd, y, warmup=2, reps=10)
        row["baseline_us"] = ts[p.info().config_index]
        row["baseline_config"] = p.info().config
        ok = [(t, n) for t, n in zip(ts, names) if t > 0]
        row["exhaustive_us"], row["exhaustive_config"] = min(ok)
        for div, key in ((1, "searched"), (0, "autotvm")):
            q = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
            r = q.search(xd, wd, sd, y, warmup=2, reps=10, trials=trials, seed=11, diversity=div)
            h = [t if t > 0 else float("inf") for t in r["history_us"]]
            row[f"{key}_us"] = r["best_us"]
            row[f"{key}_config"] = r["config"]
            row[f"{key}_curve"] = [round(v, 3) for v in np.minimum.accumulate(h).tolist()]
            row[f"{key}_failed"] = sum(t <= 0 for t in r["history_us"])
        # re-time the three picks back to back (the searches ran minutes apart)
        rows.append(row)
        print(json.dumps({k: v for k, v in row.items() if not k.endswith("_curve")}), flush=True)

json.dump({"trials": trials, "rows": rows}, open(out, "w"), indent=1)
# markdown table (Table 1 layout)
md = [f"# B200 analog of PAPER.md Table 1 (search: {trials} measurements per search)", "",
      "| layer | bits | N | TileConfigs | space points | baseline us | exhaustive us | searched us | autotvm us | "
      "speed-up (baseline/searched) | searched / exhaustive | searched config |",
      "|---|---|---|---|---|---|---|---|---|---|---|---|"]
for r in rows:
    md.append(f"| {r['layer']} | {r['bits']} | {r['N']} | {r['candidates']} | {r['space_points']} | "
              f"{r['baseline_us']:.2f} | {r['exhaustive_us']:.2f} | {r['searched_us']:.2f} | {r['autotvm_us']:.2f} | "
              f"{r['baseline_us'] / r['searched_us']:.2f}x | {r['searched_us'] / r['exhaustive_us']:.3f} | "
              f"{r['searched_config']} |")
open(os.path.splitext(out)[0] + ".md", "w").write("\n".join(md) + "\n")
print("\n".join(md))
