"""H2D bandwidth of pinned host -> device copies, 1/2/4 streams (the e2e upload of bench.py)."""
import time

import torch

n = 3_284_800_000 // 8
src = torch.empty(n, dtype=torch.float64).pin_memory()
dst = torch.empty(n, dtype=torch.float64, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = (n + ns - 1) // ns
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    print(f"{ns} streams: {n * 8 / t / 1e9:.1f} GB/s ({t * 1e3:.1f} ms)")
