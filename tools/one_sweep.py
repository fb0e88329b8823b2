"""Exactly one resident sweep after setup (for ncu launch lists / captures of the c4 path)."""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1404_0466_b200 import _lib, configs, cvsearch  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
X, Y = configs.generate(cfg)
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, configs.grid_values(cfg), g=cfg.s, r=cfg.r)
for kv in filter(None, os.environ.get("RP_OPTS", "").split(",")):  # e.g. RP_OPTS=solve_cluster=8
    k, v = kv.split("=")
    _lib.call("rp_set_option", k.encode(), int(v))
sess.upload(torch.from_numpy(X), torch.from_numpy(Y))
torch.cuda.synchronize()
sess.sweep()
torch.cuda.synchronize()
print("one sweep done")
