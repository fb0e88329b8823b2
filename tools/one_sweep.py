"""Exactly one resident sweep after setup (for ncu launch lists / captures of the c4 path)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1404_0466_b200 import configs, cvsearch  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
X, Y = configs.generate(cfg)
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, configs.grid_values(cfg), g=cfg.s, r=cfg.r)
sess.upload(torch.from_numpy(X), torch.from_numpy(Y))
torch.cuda.synchronize()
sess.sweep()
torch.cuda.synchronize()
print("one sweep done")
