"""Top instructions by warp-stall samples from an ncu report's source page."""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hdr_i]
body = [dict(zip(h, r)) for r in rows[hdr_i + 1:] if len(r) == len(h)]
tot = sum(int(b["Warp Stall Sampling (All Samples)"] or 0) for b in body)
body.sort(key=lambda b: -int(b["Warp Stall Sampling (All Samples)"] or 0))
print("total samples", tot)
for b in body[:n]:
    s = int(b["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{s:7d} {100*s/max(tot,1):5.1f}%  {b['Address'][-5:]}  {b['Source'].strip()[:90]}")
