"""Summarise an `ncu --page source --csv --print-source sass` dump: stall
reasons overall and the hottest instructions (offline helper for profiles/)."""
import csv, sys

def f(v):
    try:
        return float(v)
    except ValueError:
        return 0.0

r = list(csv.reader(open(sys.argv[1])))
h = r[1]
rows = [x for x in r[2:] if len(x) == len(h) and x[0] != "Address"]
ia, isrc = h.index("Address"), h.index("Source")
iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
sc = [i for i, c in enumerate(h) if c.startswith("stall_")]
tot = sum(f(x[iss]) for x in rows)
print("samples", tot, "warp instructions", sum(f(x[iex]) for x in rows))
agg = {}
for x in rows:
    for i in sc:
        agg[h[i]] = agg.get(h[i], 0) + f(x[i])
print({k: round(v / tot * 100, 1) for k, v in sorted(agg.items(), key=lambda t: -t[1])[:8]})
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
top = sorted(range(len(rows)), key=lambda i: -f(rows[i][iss]))[:n]
for i in sorted(top):
    x = rows[i]
    why = [(h[j][6:], int(f(x[j]))) for j in sc if f(x[j]) > 0.2 * f(x[iss])]
    print(f"{i:5d} {x[ia]:>6} {x[isrc][:58]:58s} {f(x[iss]):7.0f} {f(x[iex]):9.0f} {why}")
