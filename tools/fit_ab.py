"""A/B timing of the fit kernel (rp_fit_tiles) between library builds at a config (experiments only).

    python tools/fit_ab.py lib.so [config]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_1404_0466_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

from paper_1404_0466_b200 import configs, cvsearch  # noqa: E402

cfg = configs.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c4"]
X, Y = configs.generate(cfg)
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, configs.grid_values(cfg), g=cfg.s, r=cfg.r)
sess.upload(X, Y)
for _ in range(2):
    sess.sweep()
ts = []
for _ in range(5):
    tim = {}
    sess.sweep(timings=tim)
    ts.append(tim["fit"] * 1e3)
P = cfg.r + 1
D = cfg.d * (cfg.d + 1) / 2
gb = cfg.k * (cfg.s + P) * D * 8 / 1e9
ms = float(np.median(ts))
print(os.path.basename(sys.argv[1]), cfg.name, f"fit {ms:.3f} ms, {gb:.2f} GB algorithmic -> {gb / ms:.2f} TB/s")
