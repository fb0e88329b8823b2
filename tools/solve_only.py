"""Run one c4 sweep with a given library build (for ncu A/B of the solve kernels; experiments only)."""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_1404_0466_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

from paper_1404_0466_b200 import configs, cvsearch  # noqa: E402

cfg = configs.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c4"]
X, Y = configs.generate(cfg)
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, configs.grid_values(cfg), g=cfg.s, r=cfg.r)
sess.upload(X, Y)
sess.sweep()
torch.cuda.synchronize()
