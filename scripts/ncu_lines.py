"""Per-CUDA-source-line stall samples / instructions from an ncu report
(python scripts/ncu_lines.py rep.ncu-rep [top]): which role's code the SM time goes to."""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Line No")
i_s, i_e = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
lines, tot = [], 0
for r in rows:
    if len(r) == len(hdr) and r[0].isdigit() and r[i_s].isdigit():
        s, e = int(r[i_s]), int(r[i_e]) if r[i_e].isdigit() else 0
        lines.append((s, e, int(r[0]), r[1].strip()[:90]))
        tot += s
print(f"total samples {tot}")
for s, e, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"  {s:6d} {100 * s / max(tot, 1):5.1f}%  inst {e:9d}  L{ln:<5d} {src}")
