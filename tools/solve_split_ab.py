"""In-process A/B of the fused eval+solve plans at one config: forced single-launch chunkings
(rp_set_option("solve_lam", n)) against the planner's choice (0: at c4 the split plan, main launch of
11-lambda chunks + tail launch on the idle SMs). Times engine.stage_solve alone (CUDA events, both passes
and the tail join), alternating the variants so clock drift hits all of them alike. Experiments only.

    python tools/solve_split_ab.py [config] [lam ...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch  # noqa: E402

from paper_1404_0466_b200 import _lib, configs, cvsearch  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
variants = [int(v) for v in sys.argv[2:]] or [12, 0]
X, Y = configs.generate(cfg)
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, configs.grid_values(cfg), g=cfg.s, r=cfg.r)
if os.environ.get("NF"):  # only the first NF folds local (one wave of CTAs at smaller chunks)
    from paper_1404_0466_b200.engine import PicholEngine
    sess.engine = PicholEngine([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, cfg.q, sess.lams.shape[0], cfg.r,
                               local_folds=list(range(int(os.environ["NF"]))))
sess.upload(X, Y)
for _ in range(2):
    sess.sweep()
eng = sess.engine
res = {v: [] for v in variants}
for rnd in range(4):
    for v in variants:
        _lib.call("rp_set_option", b"solve_lam", v)
        eng.stage_solve()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            eng.stage_solve()
        e1.record()
        torch.cuda.synchronize()
        res[v].append(e0.elapsed_time(e1) / 3)
_lib.call("rp_set_option", b"solve_lam", 0)
print({v: [round(t, 2) for t in ts] for v, ts in res.items()})
print({v: round(float(np.median(ts)), 2) for v, ts in res.items()})
