"""Summarise an ncu report's source page: instruction mix per 32 outputs and the top stall sites.
python scripts/ncu_src_top.py gpurun_out/src_<layer>.ncu-rep [outputs]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
outs = float(sys.argv[2]) if len(sys.argv) > 2 else 0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]; data = rows[2:]
i_e = hdr.index("Instructions Executed"); i_s = hdr.index("Warp Stall Sampling (All Samples)")
c = collections.Counter(); s = collections.Counter(); tot = 0; stot = 0
for r in data:
    op = r[1].strip()
    if op.startswith('@'): op = op.split(None, 1)[1]
    op = op.split()[0].split('.')[0]
    c[op] += int(r[i_e]); s[op] += int(r[i_s]); tot += int(r[i_e]); stot += int(r[i_s])
print(f"warp-instructions {tot}" + (f", per 32 outputs {tot / (outs / 32):.2f}" if outs else "") + f"; stall samples {stot}")
for k, v in c.most_common(18):
    print(f"  {k:10s} {v:10d}" + (f" {v / (outs / 32):6.2f}" if outs else "") + f"  samples {s[k]}")
print("top stall sites:")
for r in sorted(data, key=lambda r: -int(r[i_s]))[:15]:
    print(f"  {r[0][-5:]} {r[i_s]:>5s} {r[i_e]:>9s}  {r[1].strip()[:70]}")
