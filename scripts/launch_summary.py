"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) of bench.py: the last complete step (quantize + the
conv launches), each launch's cold-cache time, share of the step and DRAM bytes.

python scripts/launch_summary.py gpurun_out/r01_launches.csv resnet50_int8_b256 > profiles/...txt
Also writes profiles/traffic_<workload>.json (conv DRAM bytes per step), which
bench.py reports as roofline.traffic."""
import csv
import json
import os
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402


def main(path, workload):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    ks = OrderedDict()
    for r in rows[1:]:
        d = dict(zip(h, r))
        e = ks.setdefault(d["ID"], {"name": d["Kernel Name"], "grid": d["Grid Size"], "block": d["Block Size"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    ks = list(ks.values())
    layers = {"resnet50_int8_b256": wl.resnet50_layers, "resnet18_int8_b1": wl.resnet18_layers,
              "resnet18_int4_b16": wl.resnet18_layers}[workload]()
    n = len(layers)
    # last quantize launch followed by n conv launches
    start = None
    for i in range(len(ks) - n - 1, -1, -1):
        if "quantize" in ks[i]["name"] and all("conv_igemm" in ks[i + 1 + j]["name"] for j in range(n)):
            start = i
            break
    assert start is not None, "no complete step in the launch list"
    step = ks[start:start + n + 1]
    unit = 1e-3  # gpu__time_duration.sum is in ns -> us
    tot = sum(k["gpu__time_duration.sum"] for k in step) * unit
    conv = step[1:]
    conv_t = sum(k["gpu__time_duration.sum"] for k in conv) * unit
    conv_b = sum(k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"] for k in conv)
    print(f"# ncu launch list, {workload}: last complete step = launches {start}..{start + n} of {len(ks)}")
    print("# cold-cache, serialised kernel times (ncu --clock-control none); the bench's timed step is warm and")
    print("# PDL-overlapped, so compare SHARES, not absolutes")
    print(f"{'#':>3} {'layer':10s} {'kernel (template args)':58s} {'grid':>12s} {'us':>9s} {'share':>6s} {'DRAM MB':>9s}")
    names = ["quantize"] + [L.name for L, _ in layers]
    for i, k in enumerate(step):
        nm = k["name"].replace("void convq::", "")
        nm = nm[:nm.find("(")] if "(" in nm else nm
        t = k["gpu__time_duration.sum"] * unit
        b = (k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]) / 1e6
        print(f"{i:3d} {names[i]:10s} {nm[:58]:58s} {k['grid']:>12s} {t:9.1f} {t / tot:6.1%} {b:9.1f}")
    print(f"step total {tot:.1f} us; conv_igemm_kernel {conv_t:.1f} us ({conv_t / tot:.1%} of the step), "
          f"DRAM {conv_b / 1e9:.3f} GB per step")
    out = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    json.dump({"source": os.path.basename(path), "workload": workload,
               "dram_bytes_per_step": int(conv_b), "conv_launches": n,
               "conv_kernel_us_cold": round(conv_t, 1), "step_kernel_us_cold": round(tot, 1),
               "conv_share_cold": round(conv_t / tot, 4)}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "resnet50_int8_b256")
