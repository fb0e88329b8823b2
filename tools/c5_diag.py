"""Diagnostics of the c5 device sweep against the reference's fold-0 golden (per-lambda errors)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_1404_0466_b200 import configs, cvsearch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
g = np.load(f"tests/golden/baseline_{name}.npz")
cfg = configs.CONFIGS[name]
X, Y = configs.generate(cfg)
grid = configs.grid_values(cfg)
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, grid, g=cfg.s, r=cfg.r)
curves, best = sess.run(X, Y)
ref = g["per_fold"][0]
err = np.abs(curves[0] - ref) / np.abs(ref)
pl = np.nanmax(err, axis=1)
md = g["mindiag"][0]
finite = np.isfinite(ref)
sane = np.all(finite & (ref < 100 * np.min(np.where(finite, ref, np.inf), axis=0)), axis=1)
pl = np.where(sane, pl, 0.0)
order = np.argsort(-np.nan_to_num(pl, nan=np.inf))
print("t_scale/shift", sess.t_scale, sess.t_shift, "model", g["model_info"][0])
for j in order[:25]:
    print(f"lambda idx {j} lam {grid[j]:.3e} max rel err {pl[j]:.3e} mindiag {md[j]:.3e} ref {np.nanmax(ref[j]):.3e} dev {np.nanmax(curves[0][j]):.3e}")
print("err quantiles over kept:", np.nanpercentile(pl[md >= 1e-2], [50, 90, 99, 100]))
