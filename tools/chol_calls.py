"""Per-call durations of the Cholesky kernels from a timeline file (RP_CHOL_GROUPS=1 run)."""
import sys

recs = [l.split() for l in open(sys.argv[1])]
recs = [(n, s, float(a), float(b)) for n, s, a, b in recs]
i0 = max(i for i, r in enumerate(recs) if r[0] in ("oz_holdout", "holdout_gemm") and i < len(recs) - 1)
recs = recs[i0 + 1:]
ch = [r for r in recs if r[0].startswith("chol") or r[0] in ("oz_syrk_chol", "oz_prep")][1:]
tot = {}
for n, s, a, b in ch:
    tot.setdefault(n, []).append(b - a)
for n, v in tot.items():
    print(n, len(v), "total %.2f ms" % sum(v), "first 12:", " ".join("%.3f" % x for x in v[:12]))
