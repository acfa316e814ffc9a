"""Summarise an ncu launch list of bench.py (--csv, metrics below): the last
complete step -- the input stage (s2d quantize + stem conv + max pool, or
quantize) and every conv launch -- with each launch's cold-cache time, its
share of the step, DRAM bytes, tensor-pipe utilisation and issue activity.

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,\
smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv ...
  python scripts/launch_summary.py launches.csv resnet50_int8_b256 > profiles/r02_launches_....txt

Also writes profiles/traffic_<workload>.json (conv DRAM bytes per step), which
bench.py reports as roofline.traffic."""
import csv
import json
import os
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

TENSOR = "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
ISSUE = "smsp__issue_active.avg.pct_of_peak_sustained_active"


def main(path, workload):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    ks = OrderedDict()
    for r in rows[1:]:
        d = dict(zip(h, r))
        e = ks.setdefault(d["ID"], {"name": d["Kernel Name"], "grid": d["Grid Size"], "block": d["Block Size"]})
        try:
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            pass
    ks = [k for k in ks.values() if any(t in k["name"] for t in ("conv_igemm", "quantize", "maxpool"))]
    spec = bench.workload_spec(workload)
    convs = [t[0] for t in spec.layers]
    n = len(convs)
    head = ["s2d_quantize", "conv_igemm", "maxpool"] if spec.conv1 is not None else ["quantize"]
    pattern = head + ["conv_igemm"] * n
    start = None
    for i in range(len(ks) - len(pattern), -1, -1):
        if all(pattern[j] in ks[i + j]["name"] for j in range(len(pattern))):
            start = i
            break
    assert start is not None, "no complete step in the launch list"
    step = ks[start:start + len(pattern)]
    names = (["s2d quantize", "conv1 (stem)", "maxpool"] if spec.conv1 is not None else ["quantize"]) + \
        [L.name for L in convs]
    us = [k["gpu__time_duration.sum"] * 1e-3 for k in step]
    tot = sum(us)
    conv_idx = [i for i, k in enumerate(step) if "conv_igemm" in k["name"]]
    conv_us = sum(us[i] for i in conv_idx)
    dram = [k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in step]
    conv_dram = sum(dram[i] for i in conv_idx)
    print(f"# ncu launch list ({os.path.basename(path)}), last complete step of {workload}: "
          f"{len(step)} launches, {tot:.1f} us summed (cold-cache, serialised)")
    print(f"# conv_igemm_kernel share of the step: {100 * conv_us / tot:.1f} % ({conv_us:.1f} us); "
          f"conv DRAM bytes/step {conv_dram / 1e9:.3f} GB")
    print(f"{'launch':14s} {'us':>8s} {'share%':>7s} {'DRAM MB':>9s} {'tensor%':>8s} {'issue%':>7s}  kernel")
    for nm, k, t, d in zip(names, step, us, dram):
        print(f"{nm:14s} {t:8.2f} {100 * t / tot:7.2f} {d / 1e6:9.1f} {k.get(TENSOR, float('nan')):8.1f} "
              f"{k.get(ISSUE, float('nan')):7.1f}  {k['name'][:70]}")
    out = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    with open(out, "w") as f:
        json.dump({"source": os.path.basename(path), "dram_bytes_per_step": int(conv_dram),
                   "conv_us_per_step_cold": round(conv_us, 2), "launches": len(step),
                   "conv_share_of_step": round(conv_us / tot, 4)}, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "resnet50_int8_b256")
