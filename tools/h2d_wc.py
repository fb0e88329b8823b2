"""H2D bandwidth: torch pinned (cudaHostAlloc default) vs write-combined pinned host memory."""
import ctypes
import time

import numpy as np
import torch
from cuda.bindings import runtime as cudart

n = 3_284_800_000 // 8
dst = torch.empty(n, dtype=torch.float64, device="cuda")


def bw(src):
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    return n * 8 / t / 1e9, t * 1e3


src = torch.empty(n, dtype=torch.float64).pin_memory()
src.fill_(1.0)
print("torch pinned: %.1f GB/s (%.1f ms)" % bw(src))
for flag, name in ((cudart.cudaHostAllocWriteCombined, "write-combined"), (cudart.cudaHostAllocPortable, "portable")):
    err, ptr = cudart.cudaHostAlloc(n * 8, flag)
    assert err == cudart.cudaError_t.cudaSuccess, err
    buf = (ctypes.c_double * n).from_address(ptr)
    arr = np.frombuffer(buf, dtype=np.float64)
    t = torch.from_numpy(arr)
    t.fill_(1.0)
    print(name, "is_pinned", t.is_pinned(), ": %.1f GB/s (%.1f ms)" % bw(t))
