"""Group a bench --layers-out JSON by shape: time, roofline-ideal time, gap."""
import collections, json, sys
rows = json.load(open(sys.argv[1]))["layers"]
tot = sum(r["us"] for r in rows); ideal = sum(r["us"] * r["roofline_frac"] for r in rows)
print(f"{len(rows)} layers: sum {tot:.1f} us, ideal {ideal:.1f} us")
g = collections.defaultdict(lambda: [0, 0, 0, ""])
for r in rows:
    k = r["shape"]; g[k][0] += r["us"]; g[k][1] += r["us"] * r["roofline_frac"]; g[k][2] += 1; g[k][3] = r["config"]
for k, (t, i, n, c) in sorted(g.items(), key=lambda kv: -(kv[1][0] - kv[1][1])):
    print(f"{k:24s} x{n}  {t:7.1f} us  ideal {i:6.1f}  gap {t - i:6.1f}  {c}")
