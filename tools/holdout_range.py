"""Exponent spread of the solution vectors the Gram-form hold-out multiplies (experiments): per column of
W, the largest binary exponent minus the mean exponent of the nonzeros, vs the range guard's 24 bits,
and the same for the rows of the fold Gram blocks.

    python tools/holdout_range.py [config]
"""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch  # noqa: E402

from paper_1404_0466_b200 import configs, cvsearch  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
X, Y = configs.generate(cfg)
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, configs.grid_values(cfg), g=cfg.s, r=cfg.r)
sess.upload(X, Y)
sess.sweep()
torch.cuda.synchronize()
eng = sess.engine


def spread(M):  # rows of M
    a = M.abs()
    nz = a > 0
    e = torch.where(nz, torch.floor(torch.log2(torch.where(nz, a, torch.ones_like(a)))), torch.zeros_like(a))
    mx = torch.where(nz, e, torch.full_like(e, -1e9)).amax(dim=1)
    mean = e.sum(dim=1) / nz.sum(dim=1).clamp(min=1)
    return mx - mean


q, m = cfg.q, min(cfg.m, 16)
for f in range(eng.nf):
    W = eng.W[0][f, :cfg.d, :q * m].T  # (q*m, d): one solution vector per row
    s = spread(W)
    bad = (s > 24).reshape(q, m).any(dim=1)
    lam_bad = torch.nonzero(bad).flatten().tolist()
    print(f"fold {f}: W spread max {s.max().item():.1f} bits, columns > 24 bits: {(s > 24).sum().item()} "
          f"of {q * m}; lambdas {lam_bad[:3]}..{lam_bad[-3:] if lam_bad else []} ({len(lam_bad)})")
G = eng.G[0].T  # rows of fold 0's Gram block (column-major storage)
Gl = torch.tril(G)
print(f"G_0 row spread max {spread(Gl).max().item():.1f} bits")
