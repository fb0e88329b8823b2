"""How many Gram-form hold-out columns the cancellation repair recomputes in one sweep (experiments).

    python tools/holdout_repairs.py [config]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch  # noqa: E402

from paper_1404_0466_b200 import _lib, configs, cvsearch  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
X, Y = configs.generate(cfg)
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, configs.grid_values(cfg), g=cfg.s, r=cfg.r)
sess.upload(X, Y)
sess.sweep()
torch.cuda.synchronize()
eng = sess.engine
n_val, d, N, nf = cfg.n // cfg.k, cfg.d, cfg.q * min(cfg.m, 16), eng.nf
mt = max((n_val + 127) // 128, 2 * ((d + 127) // 128))
off = (8 * (nf * mt * N + nf * N) + 1023) // 1024 * 1024
count = int(eng.ws_hold[off:off + 4].view(torch.int32).item())
_lib.call("rp_set_option", b"profile", 1)
_lib.query("rp_profile_ms", None)
tim = {}
sess.sweep(timings=tim)
print(f"{cfg.name}: repaired columns {count} of {nf * N} ({100.0 * count / (nf * N):.1f}%), "
      f"hold-out stage {tim['predict_local'] * 1e3:.2f} ms")
