"""Per-kernel totals of an ncu launch list (`--metrics gpu__time_duration.sum --csv`) as markdown rows.

    python tools/launch_summary.py profiles/r01_launches_c4_sweep.csv
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
tot = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    name = r[ki].split("(")[0]
    tot[name][0] += 1
    tot[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
T = sum(t for _, t in tot.values())
print(f"{sum(c for c, _ in tot.values())} launches, {T:.2f} ms serialised")
for n, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"| `{n}` | {c} | {t:.2f} | {100 * t / T:.1f}% |")
