"""Per-stage sweep times (median of 5, CUDA events between stages) for one library build and the current
environment switches (experiments only).

    RP_CHOL_GROUPS=8 python tools/stage_ab.py [lib.so] [config]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_1404_0466_b200 import _lib  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    _lib.LIB_PATH = os.path.abspath(sys.argv.pop(1))
import torch  # noqa: E402

from paper_1404_0466_b200 import configs, cvsearch  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
X, Y = configs.generate(cfg)
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, configs.grid_values(cfg), g=cfg.s, r=cfg.r)
sess.upload(X, Y)
for _ in range(2):
    sess.sweep()
res = {}
for _ in range(5):
    tim = {}
    sess.sweep(timings=tim)
    for k, v in tim.items():
        res.setdefault(k, []).append(v * 1e3)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    sess.sweep()
e1.record()
torch.cuda.synchronize()
env = {k: v for k, v in os.environ.items() if k.startswith("RP_")}
print(env, {k: round(float(np.median(v)), 2) for k, v in res.items()}, "sweep", round(e0.elapsed_time(e1) / 5, 2))
