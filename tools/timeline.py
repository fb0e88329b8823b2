"""Kernel timeline of one resident c4 sweep (CUDA events around each profiled launch, every stream):
per-kernel totals and, for the factorization window, how busy each stream group is. Diagnostic."""
import collections
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1404_0466_b200 import _lib, configs, cvsearch  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/timeline.txt"
X, Y = configs.generate(cfg)
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, configs.grid_values(cfg), g=cfg.s, r=cfg.r)
sess.upload(torch.from_numpy(X), torch.from_numpy(Y))
for _ in range(2):
    sess.sweep()
torch.cuda.synchronize()
os.environ["RP_PROF_TIMELINE"] = out
_lib.call("rp_set_option", b"profile", 1)
_lib.query("rp_profile_ms", None)
sess.sweep()
sess.sweep()  # analysed: the second of two back-to-back sweeps (clocks already up)
_lib.query("rp_profile_ms", None)
_lib.call("rp_set_option", b"profile", 0)
recs = [l.split() for l in open(out)]
recs = [(n, s, float(a), float(b)) for n, s, a, b in recs]
second = [i for i, r in enumerate(recs) if r[0] == recs[0][0]][1]  # the second sweep's first record
recs = recs[second:]
t00 = recs[0][2]
recs = [(n, s, a - t00, b - t00) for n, s, a, b in recs]
tot = collections.defaultdict(lambda: [0, 0.0])
for n, s, a, b in recs:
    tot[n][0] += 1
    tot[n][1] += b - a
print("kernel totals (ms, serial sum of event windows):")
for n, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"  {n:16s} {c:5d} launches {t:8.2f} ms")
ch = [r for r in recs if r[0].startswith("chol") or r[0] == "oz_syrk_chol" or (r[0] == "oz_prep" and r[2] > 0)]
chol = [r for r in recs if r[0].startswith("chol")]
if chol:
    t0 = min(r[2] for r in chol)
    t1 = max(r[3] for r in recs if r[0] in ("chol_trsm", "chol_diag", "chol_update", "oz_syrk_chol"))
    print(f"factorization window {t0:.2f} -> {t1:.2f} = {t1 - t0:.2f} ms")
    by = collections.defaultdict(list)
    for r in recs:
        if r[2] >= t0 - 1e-3 and r[3] <= t1 + 1e-3:
            by[r[1]].append(r)
    for s, rs in by.items():
        busy = sum(b - a for _, _, a, b in rs)
        names = collections.Counter(r[0] for r in rs)
        per = {n: round(sum(b - a for m, _, a, b in rs if m == n), 2) for n in names}
        print(f"  stream {s}: {len(rs)} launches, busy {busy:.2f} ms of {t1 - t0:.2f}: {per}")
