"""One batched Cholesky of c4-sized matrices (experiments: ncu captures of the factorization kernels)."""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1404_0466_b200 import _dev, _ops  # noqa: E402

d, batch = 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 10
rng = np.random.default_rng(0)
B = rng.standard_normal((d, d)) * 0.01
M = B @ B.T + np.eye(d)
A = _dev.to_dev(np.tile(np.ascontiguousarray(M.T).reshape(-1), batch))
info = _ops.potrf(A, d, batch)
torch.cuda.synchronize()
print("info", info.max())
