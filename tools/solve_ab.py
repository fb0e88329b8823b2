"""A/B timing of the fused eval+solve between two builds of the library (experiments only).

    python tools/solve_ab.py path/to/libridgepath_b200.so [config]
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
grid = configs.grid_values(cfg)
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, grid, g=cfg.s, r=cfg.r)
for kv in filter(None, os.environ.get("RP_OPTS", "").split(",")):  # e.g. RP_OPTS=solve_cluster=2
    k, v = kv.split("=")
    _lib.call("rp_set_option", k.encode(), int(v))
sess.upload(X, Y)
for _ in range(3):
    sess.sweep()
torch.cuda.synchronize()
_lib.call("rp_set_option", b"profile", 1)
res = {}
for rep in range(5):
    _lib.query("rp_profile_ms", None)
    sess.sweep()
    for n in ("eval_solve", "eval_solve_fwd", "eval_solve_bwd", "oz_syrk"):
        res.setdefault(n, []).append(_lib.query("rp_profile_ms", n.encode()))
    res.setdefault("all", []).append(_lib.query("rp_profile_ms", None))
print(os.path.basename(sys.argv[1]), os.environ.get("RP_OPTS", ""), {k: round(float(np.median(v)), 3) for k, v in res.items()})
