"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
the profiles/ text format: per-kernel counts and totals, and the shares of the
Projected-Adam step kernels. usage: launch_summary.py launches.csv header-line"""
import csv
import io
import sys
from collections import defaultdict

rows = [r for r in csv.reader(io.StringIO("".join(l for l in open(sys.argv[1]) if l.startswith('"'))))]
head, data = rows[0], rows[1:]
ik, iv, iu = head.index("Kernel Name"), head.index("Metric Value"), head.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
for r in data:
    v = float(r[iv].replace(",", ""))
    v = v / 1e6 if r[iu] == "ns" else v / 1e3 if r[iu] in ("us", "usecond") else v
    name = r[ik].split("(")[0][:62]
    tot[name] += v
    cnt[name] += 1
print(sys.argv[2] if len(sys.argv) > 2 else "# ncu launch list")
print("# cold-cache serialised launch times (ncu); compare shares, not absolutes.")
print(f"{'kernel':62s} {'count':>6s} {'total_ms':>12s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:62s} {cnt[k]:6d} {tot[k]:12.3f}")
step = {k: v for k, v in tot.items() if "k_apply" in k or "k_transpose" in k}
s = sum(step.values())
print("\n# share of the Projected-Adam step (k_apply + k_transpose):")
for k, v in step.items():
    print(f"{k:62s} {100 * v / s:5.1f}%  avg {v / cnt[k]:.3f} ms/launch")
