"""Solve time of the c4 sweep for a subset of local folds (the per-rank work at N GPUs)."""
import os
import sys

sys.path.insert(0, ".")
from paper_1404_0466_b200 import _lib  # noqa: E402

if os.environ.get("RP_LIB"):  # A/B of library builds
    _lib.LIB_PATH = os.path.abspath(os.environ["RP_LIB"])
import torch  # noqa: E402

from paper_1404_0466_b200 import _lib, configs, cvsearch, dist  # noqa: E402

cfg = configs.CONFIGS["c4"]
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
X, Y = configs.generate(cfg)
shard = dist.Shard(0, world, cfg.k)
shard_local = dist.Shard(0, world, cfg.k)
for kv in filter(None, os.environ.get("RP_OPTS", "").split(",")):  # e.g. RP_OPTS=solve_cluster=8
    k, v = kv.split("=")
    _lib.call("rp_set_option", k.encode(), int(v))
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, configs.grid_values(cfg), g=cfg.s, r=cfg.r)
# emulate rank 0 of `world`: only its folds are local (all Gram blocks computed here, no exchange)
from paper_1404_0466_b200.engine import PicholEngine  # noqa: E402
eng = PicholEngine([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, cfg.q, sess.lams.shape[0], cfg.r,
                   local_folds=shard.local_folds)
sess.engine = eng
sess.upload(torch.from_numpy(X), torch.from_numpy(Y))
for _ in range(2):
    sess.sweep()
tim = {}
for _ in range(3):
    tim.clear()
    sess.sweep(timings=tim)
_lib.call("rp_set_option", b"profile", 1)
_lib.query("rp_profile_ms", None)
sess.sweep()
solve = _lib.query("rp_profile_ms", b"eval_solve_fwd") + _lib.query("rp_profile_ms", b"eval_solve_bwd")
_lib.call("rp_set_option", b"profile", 0)
print(f"opts={os.environ.get('RP_OPTS', '')} world={world} local={shard.local_folds} stages(ms)={ {k: round(v * 1e3, 2) for k, v in tim.items()} } solve_kernel={solve:.2f}")
