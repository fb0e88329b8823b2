"""Timeline of the end-to-end c4 run (pinned host X/Y streamed per fold block): when each block's
copy lands and when each device stage ends, relative to the first copy. Diagnostic only."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1404_0466_b200 import configs, cvsearch  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
X, Y = configs.generate(cfg)
grid = configs.grid_values(cfg)
sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, grid, g=cfg.s, r=cfg.r)
Xp = torch.from_numpy(X).pin_memory()
Yp = torch.from_numpy(Y).pin_memory()
for _ in range(2):
    sess.run(Xp, Yp)
torch.cuda.synchronize()
# plain H2D of X
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sess.X.copy_(Xp, non_blocking=True)
    torch.cuda.synchronize()
    print(f"H2D X alone: {(time.perf_counter() - t0) * 1e3:.1f} ms ({Xp.numel() * 8 / (time.perf_counter() - t0) / 1e9:.1f} GB/s)")
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sess.run(Xp, Yp)
    print(f"run(): {(time.perf_counter() - t0) * 1e3:.1f} ms")
# timeline
eng = sess.engine
torch.cuda.synchronize()
t0 = time.perf_counter()
start = torch.cuda.Event(enable_timing=True)
start.record()
cs = sess._copy_stream
cs.wait_stream(torch.cuda.current_stream())
ready = {}
with torch.cuda.stream(cs):
    sess.Y.copy_(Yp, non_blocking=True)
    for b in range(eng.k):
        lo, hi = int(eng.row_off[b]), int(eng.row_off[b + 1])
        sess.X[lo:hi].copy_(Xp[lo:hi], non_blocking=True)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(cs)
        ready[b] = ev
tim = {}
curves, _, best = eng.sweep(sess.X, sess.Y, sess.lams, sess.P, sess.V, sess.tvals, timings=tim, block_ready=ready)
t_host_enq = time.perf_counter() - t0
torch.cuda.synchronize()
t_dev = time.perf_counter() - t0
print("block copies done at", [round(start.elapsed_time(ready[b]), 1) for b in range(eng.k)])
print(f"host enqueue {t_host_enq * 1e3:.1f} ms, sync at {t_dev * 1e3:.1f} ms; stage durations {dict((k, round(v * 1e3, 2)) for k, v in tim.items())}")
t1 = time.perf_counter()
bad = eng.check_numerics(sess.lams)
c = curves.cpu().numpy(); b = best.cpu().numpy()
print(f"readback {(time.perf_counter() - t1) * 1e3:.1f} ms")

# per-stage timeline (both streams): wrap the engine's stage methods with events on the current stream
recs = []
for name in ("stage_gram", "stage_systems", "stage_factorize", "stage_fit", "stage_solve", "stage_holdout",
             "stage_select"):
    fn = getattr(eng, name)

    def wrapped(*a, _fn=fn, _name=name, **kw):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        out = _fn(*a, **kw)
        e1.record()
        recs.append((_name, kw.get("part", a[-1] if a and isinstance(a[-1], tuple) else None),
                     torch.cuda.current_stream().stream_id, e0, e1))
        return out
    setattr(eng, name, wrapped)
for rep in range(2):
    recs.clear()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    start.record()
    sess.run(Xp, Yp)
    torch.cuda.synchronize()
    end = torch.cuda.Event(enable_timing=True)
print("timeline (ms from start):")
for name, part, sid, e0, e1 in recs:
    print(f"  {name:16s} part={part} stream={sid}: {start.elapsed_time(e0):7.2f} -> {start.elapsed_time(e1):7.2f}")
