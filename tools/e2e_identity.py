"""Full-size check: the end-to-end session (pinned host X/Y streamed per block) returns curves
bit-identical to the device-resident sweep of the same session (c4 by default)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1404_0466_b200 import configs, cvsearch  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
X, Y = configs.generate(cfg)
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, configs.grid_values(cfg), g=cfg.s, r=cfg.r)
c_stream, b_stream = sess.run(torch.from_numpy(X).pin_memory(), torch.from_numpy(Y).pin_memory())
c_res, b_res = sess.run(X, Y)
print(cfg.name, "bit-identical:", np.array_equal(c_stream, c_res), np.array_equal(b_stream, b_res),
      "best:", b_res.tolist())
