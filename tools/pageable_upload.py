"""Upload of a pageable numpy design (the drop-in grid_search_pichol input) to the device: torch's pageable
copy vs a staged pipeline (worker threads copy row chunks into pinned slots while the previous chunk's DMA
runs) vs page-locking the numpy buffer in place (cudaHostRegister). Experiments only.

    python tools/pageable_upload.py [n] [d]
"""
import concurrent.futures as cf
import sys
import time

import numpy as np
import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
X = np.full((n, d), 1.5)
X[::7] = 2.5
dst = torch.empty((n, d), dtype=torch.float64, device="cuda")
gb = X.nbytes / 1e9


def t_pageable():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dst.copy_(torch.from_numpy(X), non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


def make_staged(chunk_mb, nslots, nthreads):
    rows = max(1, int(chunk_mb * 2**20) // (d * 8))
    slots = [torch.empty((rows, d), dtype=torch.float64).pin_memory() for _ in range(nslots)]
    views = [s.numpy() for s in slots]
    evs = [None] * nslots
    cs = torch.cuda.Stream()
    pool = cf.ThreadPoolExecutor(nthreads)

    def run():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for c, lo in enumerate(range(0, n, rows)):
            hi = min(n, lo + rows)
            k = c % nslots
            if evs[k] is not None:
                evs[k].synchronize()
            part = (hi - lo + nthreads - 1) // nthreads
            futs = [pool.submit(np.copyto, views[k][a - lo:min(hi, a + part) - lo], X[a:min(hi, a + part)])
                    for a in range(lo, hi, part)]
            for f in futs:
                f.result()
            with torch.cuda.stream(cs):
                dst[lo:hi].copy_(slots[k][: hi - lo], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
                evs[k] = ev
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    return run


def t_register():
    cr = torch.cuda.cudart()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = cr.cudaHostRegister(X.ctypes.data, X.nbytes, 0)
    t1 = time.perf_counter()
    src = torch.from_numpy(X)
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cr.cudaHostUnregister(X.ctypes.data)
    t3 = time.perf_counter()
    return rc, t1 - t0, t2 - t1, t3 - t2


for rep in range(2):
    t = t_pageable()
    print(f"pageable copy_: {t * 1e3:.1f} ms ({gb / t:.1f} GB/s)")
for chunk_mb, nslots, nth in ((32, 3, 4), (64, 3, 4), (64, 3, 8), (128, 3, 8), (32, 4, 8), (256, 2, 8)):
    run = make_staged(chunk_mb, nslots, nth)
    ts = [run() for _ in range(3)]
    t = min(ts)
    print(f"staged chunk {chunk_mb} MB x {nslots} slots, {nth} threads: {t * 1e3:.1f} ms ({gb / t:.1f} GB/s)")
for rep in range(2):
    rc, a, b, c = t_register()
    print(f"cudaHostRegister rc={rc}: register {a * 1e3:.1f} ms, DMA {b * 1e3:.1f} ms ({gb / b:.1f} GB/s), "
          f"unregister {c * 1e3:.1f} ms")
