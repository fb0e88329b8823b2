"""Cross-validated selection of the ridge parameter on the B200
(drop-in for the hot path of ridgepath/cvsearch.py).

``grid_search_pichol`` (cvsearch.py:206-243) keeps the reference's signature,
validation and report (CvReport with per-lambda fold-mean errors keyed by
float(lambda), first-argmin selection, per-fold CSV rows and phase timings).
The whole sweep -- per-fold Hessians, the s x k sampled-lambda Choleskys, the
polynomial fit, the fused evaluate+solve for all q lambdas and the hold-out
errors -- runs on the device through ``engine.PicholEngine``; only the q x m
curve matrix and the selection come back to the host.

Multi-output generalization: ``Dataset.y`` may be (n, m). The per-output fold
curves are in ``CvReport.curves`` (k, q, m) with per-output selections in
``best_index``; ``per_lambda_error``/``best_lambda``/``best_error`` then
describe the mean over outputs. For 1-D y the report matches the reference.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _ops, pichol, trivec
from .engine import MISCLASS, RMSE, PicholEngine
from .errors import DimensionMismatch, EmptyValidationSet, InvalidThreshold, SingularInterpolant, UsageError

METRICS = (RMSE, MISCLASS)
PHASES = ("factorize", "vec", "fit", "interp", "solve", "predict")
THREADS_ENV = "RIDGEPATH_THREADS"


@dataclass
class Dataset:
    """Full design and labels; fold plans slice it into train/validation."""

    X: np.ndarray
    y: np.ndarray


@dataclass
class LambdaGrid:
    lo: float
    hi: float
    q: int
    values: np.ndarray


def make_grid(lo, hi, q):
    """q log-spaced values from lo to hi inclusive (cvsearch.py:55-66)."""
    if not (0 < lo < hi):
        raise UsageError(f"need 0 < lo < hi, got lo={lo}, hi={hi}")
    if q < 1:
        raise UsageError(f"grid size must be >= 1, got q={q}")
    if q == 1:
        values = np.array([lo])
    else:
        values = np.logspace(np.log10(lo), np.log10(hi), q)
        values[0], values[-1] = lo, hi
    return LambdaGrid(lo=lo, hi=hi, q=q, values=values)


@dataclass
class FoldPlan:
    k: int
    assignments: np.ndarray
    seed: int


def make_folds(n, k, seed, labels=None):
    """Seeded fold assignment; stratified when labels are +/-1 (cvsearch.py:76-92)."""
    if k < 2:
        raise UsageError(f"need k >= 2 folds, got {k}")
    if k > n:
        raise UsageError(f"cannot split {n} samples into {k} nonempty folds")
    rng = np.random.default_rng(seed)
    assignments = np.empty(n, dtype=np.int64)
    if labels is not None and set(np.unique(labels)) <= {-1.0, 1.0}:
        for cls in (-1.0, 1.0):
            idx = np.flatnonzero(np.asarray(labels) == cls)
            idx = rng.permutation(idx)
            assignments[idx] = np.arange(idx.size) % k
    else:
        perm = rng.permutation(n)
        assignments[perm] = np.arange(n) % k
    return FoldPlan(k=k, assignments=assignments, seed=seed)


def contiguous_folds(n, k, seed=0):
    """BASELINE.json folds: contiguous blocks of n // k rows."""
    return FoldPlan(k=k, assignments=np.arange(n) // (n // k), seed=seed)


@dataclass
class CvReport:
    method: str
    per_lambda_error: dict
    best_lambda: float
    best_error: float
    timings: dict
    rows: list = field(default_factory=list)
    wall_seconds: float = 0.0
    curves: np.ndarray | None = None  # (k, q, m) per-fold, per-output errors
    best_index: np.ndarray | None = None  # (m,) per-output first-argmin index


def holdout_error(theta, X_val, y_val, metric=RMSE):
    """Validation error of one solution (cvsearch.py:106-123), computed on the device."""
    X_val = np.asarray(X_val, dtype=float)
    y_val = np.asarray(y_val, dtype=float).reshape(-1)
    if X_val.shape[0] == 0:
        raise EmptyValidationSet("validation set is empty")
    if X_val.shape[0] != y_val.shape[0]:
        raise DimensionMismatch(f"{X_val.shape[0]} rows vs {y_val.shape[0]} targets")
    if metric not in METRICS:
        raise UsageError(f"unknown metric {metric!r}")
    return float(_ops.holdout(np.asarray(theta, dtype=float).reshape(-1), X_val, y_val, metric)[0])


def resolve_threads(threads=None):
    """Thread count from the argument, RIDGEPATH_THREADS, or 1 (cvsearch.py:126-134).

    Accepted for API compatibility; the device sweep does not use host threads."""
    if threads is None:
        threads = os.environ.get(THREADS_ENV, "1")
    try:
        threads = int(threads)
    except ValueError as e:
        raise UsageError(f"bad thread count {threads!r}") from e
    return max(1, threads)


def _zero_timings():
    return dict.fromkeys(PHASES, 0.0)


def fold_order(folds, n):
    """Stable grouping of rows by fold (keeps the reference's row order inside each fold,
    cvsearch.py:145-147). Returns (row order, rows per fold)."""
    a = np.asarray(folds.assignments)
    if a.shape[0] != n:
        raise DimensionMismatch(f"fold plan covers {a.shape[0]} rows, data has {n}")
    counts = np.bincount(a, minlength=folds.k)[: folds.k]
    if np.any(a < 0) or np.any(a >= folds.k):
        raise UsageError("fold assignments outside [0, k)")
    if np.any(counts == 0):
        raise EmptyValidationSet("validation set is empty")
    if np.all(a[:-1] <= a[1:]):
        return None, counts
    return np.argsort(a, kind="stable"), counts


def _merge(method, grid_values, curves, times_per_fold, wall):
    """Fold mean + first argmin + CSV rows (cvsearch.py:154-175). curves: (k, q, m)."""
    k, q, m = curves.shape
    errs_all = np.mean(curves, axis=0)  # (q, m)
    errs = errs_all[:, 0] if m == 1 else np.mean(errs_all, axis=1)
    timings = _zero_timings()
    rows = []
    for i in range(k):
        for phase in PHASES:
            timings[phase] += times_per_fold[phase]
        fold_errs = curves[i, :, 0] if m == 1 else np.mean(curves[i], axis=1)
        for lam, e in zip(grid_values, fold_errs):
            rows.append({"fold": i, "lambda": float(lam), "error": float(e), **times_per_fold})
    best_idx = int(np.argmin(errs))
    for lam, e in zip(grid_values, errs):
        rows.append({"fold": -1, "lambda": float(lam), "error": float(e), **_zero_timings()})
    return CvReport(
        method=method,
        per_lambda_error={float(l): float(e) for l, e in zip(grid_values, errs)},
        best_lambda=float(grid_values[best_idx]),
        best_error=float(errs[best_idx]),
        timings=timings,
        rows=rows,
        wall_seconds=wall,
        curves=curves,
        best_index=np.argmin(errs_all, axis=0),
    )


def prepare_design(p, folds):
    """Host arrays grouped by fold (no copy for contiguous plans): (X, Y (n, m), block rows)."""
    X = np.asarray(p.X, dtype=float)
    y = np.asarray(p.y, dtype=float)
    Y = y.reshape(-1, 1) if y.ndim == 1 else y
    if X.ndim != 2 or X.shape[0] != Y.shape[0]:
        raise DimensionMismatch(f"{X.shape[0]} rows vs {Y.shape[0]} targets")
    order, counts = fold_order(folds, X.shape[0])
    if order is not None:
        X, Y = X[order], Y[order]
    return np.ascontiguousarray(X), np.ascontiguousarray(Y), counts


class CvSession:
    """A reusable device-resident piCholesky CV sweep for fixed shapes and grid.

    The public entry point behind ``grid_search_pichol`` and the end-to-end bench:
    ``run(X, Y)`` takes host arrays (numpy, or pinned torch tensors for an async
    copy), moves them to the device, runs the sweep and returns the curves.
    block_rows are the rows per fold block with X/Y grouped by fold.
    With a ``dist.Shard`` the session computes its local folds and exchanges
    Gram blocks and curves over torch.distributed.
    """

    STAGE_BYTES = 256 << 20  # each of the two pinned staging slots of upload_pageable

    def __init__(self, block_rows, d, m, grid_values, g=4, r=2, metric=RMSE, holdout="auto",
                 raw_monomials=False, shard=None):
        import torch

        from . import dist

        grid_values = np.asarray(grid_values, dtype=float)
        q = grid_values.shape[0]
        if g > q:
            raise UsageError(f"cannot draw g={g} samples from a grid of {q}")
        self.grid = grid_values
        self.sample_lams = grid_values[pichol.sample_indices(q, g)]
        self.lams, self.V, self.cond_V, self.t_scale, self.t_shift, self.P = _fit_basis_checked(
            self.sample_lams, r, raw_monomials)
        self.shard = shard
        kw = {}
        if shard is not None:
            kw = dict(local_folds=shard.local_folds, gram_blocks=shard.gram_blocks)
        self.engine = PicholEngine(block_rows, d, m, q, self.lams.shape[0], r, metric=metric, holdout=holdout, **kw)
        eng = self.engine
        self.X = torch.empty((eng.n, d), dtype=torch.float64, device=eng.device)
        self.Y = torch.empty((eng.n, m), dtype=torch.float64, device=eng.device)
        self.tvals = _dev.to_dev(self.t_scale * grid_values + self.t_shift)
        self._exchange = None
        self._gather = None
        self._copy_stream = None
        if shard is not None and shard.world > 1:
            self._exchange = lambda e: dist.exchange_grams(shard, e.G, e.C, e.yy)
            self._gather = lambda c: dist.gather_curves(shard, c)

    @property
    def needed_blocks(self):
        """Row blocks this device reads (all of them without a shard; a rank's own blocks when the
        Gram blocks are exchanged)."""
        return self.shard.needed_blocks if self.shard is not None else list(range(self.engine.k))

    @property
    def h2d_bytes(self):
        eng = self.engine
        rows = sum(int(eng.row_off[b + 1] - eng.row_off[b]) for b in self.needed_blocks)
        return rows * (eng.d + eng.m) * 8

    @property
    def d2h_bytes(self):
        e = self.engine
        return e.k * e.q * e.m * 8 + e.m * 4 + e.info.numel() * 4 + e.flags.numel() * 4

    def upload(self, X, Y):
        import torch

        eng = self.engine
        blocks = self.needed_blocks
        whole = len(blocks) == eng.k
        for dst, src in ((self.X, X), (self.Y, Y)):
            if not isinstance(src, torch.Tensor):
                src = torch.from_numpy(np.ascontiguousarray(src, dtype=np.float64))
            src = src.reshape(dst.shape)
            if whole:
                dst.copy_(src, non_blocking=True)
                continue
            for b in blocks:  # only the rows this rank reads
                lo, hi = int(eng.row_off[b]), int(eng.row_off[b + 1])
                dst[lo:hi].copy_(src[lo:hi], non_blocking=True)

    def upload_streamed(self, X, Y):
        """Copy pinned host X/Y fold block by fold block on a side stream; returns the per-block
        events the Gram stage waits on (the copy of block b+1 overlaps the Gram of block b)."""
        return self._upload_into(self.X, self.Y, X, Y, None)

    def _upload_into(self, Xd, Yd, X, Y, buffer_free):
        """Per-block copies of pinned host X/Y into the device buffers Xd/Yd on the copy stream, after
        `buffer_free` (an event: the last sweep that read Xd/Yd finished; None: everything enqueued so
        far on the current stream). Returns {block: event}."""
        import torch

        eng = self.engine
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream()
        cs = self._copy_stream
        if buffer_free is None:
            cs.wait_stream(torch.cuda.current_stream())  # previous users of X/Y are done
        else:
            cs.wait_event(buffer_free)
        ready = {}
        with torch.cuda.stream(cs):
            needed = self.needed_blocks
            Yh = Y.reshape(Yd.shape)
            order = [b for b in eng.gram_blocks if b in needed] + [b for b in needed if b not in eng.gram_blocks]
            for b in order:
                lo, hi = int(eng.row_off[b]), int(eng.row_off[b + 1])
                Yd[lo:hi].copy_(Yh[lo:hi], non_blocking=True)
            for b in order:
                lo, hi = int(eng.row_off[b]), int(eng.row_off[b + 1])
                Xd[lo:hi].copy_(X[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
                ready[b] = ev
        return ready

    def upload_pageable(self, X, Y):
        """Pageable host X/Y (numpy): worker threads copy row chunks into two pinned staging slots while
        the previous chunk's DMA runs on the copy stream (torch's own pageable copy moves ~11 GB/s; this
        ~45 GB/s at c4, tools/pageable_upload.py). Returns {block: callable}: calling one copies that
        block and returns its event, so the engine starts each block's upload right before its Gram and
        the host copy of block b+1 overlaps the Gram of block b."""
        import concurrent.futures as cf

        import torch

        eng = self.engine
        X = np.ascontiguousarray(X, dtype=np.float64).reshape(tuple(self.X.shape))
        Y = np.ascontiguousarray(Y, dtype=np.float64).reshape(tuple(self.Y.shape))
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream()
        cs = self._copy_stream
        cs.wait_stream(torch.cuda.current_stream())  # previous users of X/Y are done
        d = eng.d
        if getattr(self, "_stage", None) is None:
            rows = max(1, min(eng.n, self.STAGE_BYTES // (8 * d)))
            slots = [torch.empty((rows, d), dtype=torch.float64).pin_memory() for _ in range(2)]
            self._stage = dict(rows=rows, slots=slots, views=[t.numpy() for t in slots], done=[None, None],
                               next=0, pool=cf.ThreadPoolExecutor(max(1, min(8, os.cpu_count() or 1))),
                               y=torch.empty(tuple(self.Y.shape), dtype=torch.float64).pin_memory())
        stg = self._stage
        workers = stg["pool"]._max_workers
        np.copyto(stg["y"].numpy(), Y)
        with torch.cuda.stream(cs):
            self.Y.copy_(stg["y"], non_blocking=True)
        y_done = torch.cuda.Event()
        y_done.record(cs)

        def copy_rows(lo, hi):
            k = stg["next"]
            stg["next"] = 1 - k
            if stg["done"][k] is not None:
                stg["done"][k].synchronize()  # the slot's previous DMA has read it
            view = stg["views"][k]
            part = -(-(hi - lo) // workers)
            futs = [stg["pool"].submit(np.copyto, view[a - lo:min(hi, a + part) - lo], X[a:min(hi, a + part)])
                    for a in range(lo, hi, part)]
            for f in futs:
                f.result()
            with torch.cuda.stream(cs):
                self.X[lo:hi].copy_(stg["slots"][k][:hi - lo], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
            stg["done"][k] = ev
            return ev

        def block(b):
            lo, hi = int(eng.row_off[b]), int(eng.row_off[b + 1])
            ev = y_done
            for a in range(lo, hi, stg["rows"]):
                ev = copy_rows(a, min(hi, a + stg["rows"]))
            return ev

        return {b: (lambda b=b: block(b)) for b in self.needed_blocks}

    def run_stream(self, pairs):
        """Host in, host out for a sequence of (X, Y) pinned host tensors of this session's shapes
        (several targets or datasets on one design shape): yields (curves, best index) per pair, in
        order. The upload of pair i+1 goes into a second device buffer on the copy stream while pair
        i's sweep runs, so in steady state the PCIe transfer hides behind the previous sweep; each
        sweep's Gram still waits block by block for its own upload, and each result is read back to
        the host before it is yielded. The read-back is asynchronous (pinned result buffers, one per
        parity): pair i's result is awaited only after pair i+1's sweep has been enqueued, so the device
        never idles while the host launches the next sweep (a failure of pair i therefore surfaces when
        its result is yielded, after pair i+1 was started)."""
        import torch

        if not hasattr(self, "_X2"):
            self._X2 = torch.empty_like(self.X)
            self._Y2 = torch.empty_like(self.Y)
        bufs = [(self.X, self.Y), (self._X2, self._Y2)]
        free = [None, None]
        it = iter(pairs)
        cur = next(it, None)
        if cur is None:
            return
        for t in cur:
            if not (isinstance(t, torch.Tensor) and t.is_pinned()):
                raise UsageError("run_stream takes pinned host torch tensors (X, Y)")
        ready = self._upload_into(bufs[0][0], bufs[0][1], cur[0], cur[1], None)
        i = 0
        pending = None
        while cur is not None:
            b = i % 2
            cur_ready = ready
            nxt = next(it, None)
            if nxt is not None:  # overlaps the sweep below
                ready = self._upload_into(bufs[1 - b][0], bufs[1 - b][1], nxt[0], nxt[1], free[1 - b])
            curves, _, best = self.engine.sweep(bufs[b][0], bufs[b][1], self.lams, self.P, self.V, self.tvals,
                                                exchange_grams=self._exchange, gather_curves=self._gather,
                                                block_ready=cur_ready)
            done = torch.cuda.Event()
            done.record()
            free[b] = done
            snap = self._read_back_async(curves, best, b)
            if pending is not None:
                yield self._await_result(pending)
            pending = snap
            cur = nxt
            i += 1
        if pending is not None:
            yield self._await_result(pending)

    def _read_back_async(self, curves, best, parity):
        """Stream-ordered copies of a sweep's results (curves, selection, Cholesky info, singular flags) into
        this parity's pinned host buffers; returns (event, buffers)."""
        import torch

        eng = self.engine
        if not hasattr(self, "_res"):
            self._res = [None, None]
        src = (curves, best, eng.info, eng.flags.amax(dim=0))
        if self._res[parity] is None or any(h.shape != t.shape for h, t in zip(self._res[parity], src)):
            self._res[parity] = tuple(torch.empty(tuple(t.shape), dtype=t.dtype).pin_memory() for t in src)
        for h, t in zip(self._res[parity], src):
            h.copy_(t, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return ev, self._res[parity]

    def _await_result(self, snap):
        ev, (curves, best, info, flags) = snap
        ev.synchronize()
        bad = self.engine.check_numerics(self.lams, info=info.numpy(), flags=flags.numpy())
        if bad is not None:
            f, j = bad
            raise SingularInterpolant(f"interpolated factor is singular at lambda={self.grid[j]} (fold {f})")
        return curves.numpy().copy(), best.numpy().copy()

    def sweep(self, timings=None, block_ready=None):
        """Device-only sweep on the resident X/Y; returns device (curves, mean, best)."""
        return self.engine.sweep(self.X, self.Y, self.lams, self.P, self.V, self.tvals,
                                 exchange_grams=self._exchange, gather_curves=self._gather, timings=timings,
                                 block_ready=block_ready)

    def run(self, X, Y, timings=None):
        """Host in, host out: (curves (k, q, m), best index (m,)) as numpy.

        Pinned torch tensors are streamed in per fold block, overlapped with the Gram stage; pageable
        arrays go through pinned staging slots the same way (upload_pageable)."""
        import torch

        pinned = isinstance(X, torch.Tensor) and X.is_pinned() and isinstance(Y, torch.Tensor) and Y.is_pinned()
        if pinned:
            ready = self.upload_streamed(X, Y)
            curves, _, best = self.engine.sweep(self.X, self.Y, self.lams, self.P, self.V, self.tvals,
                                                exchange_grams=self._exchange, gather_curves=self._gather,
                                                timings=timings, block_ready=ready)
        elif isinstance(X, torch.Tensor) or isinstance(Y, torch.Tensor):
            self.upload(X, Y)
            curves, _, best = self.sweep(timings)
        else:
            ready = self.upload_pageable(X, Y)
            curves, _, best = self.engine.sweep(self.X, self.Y, self.lams, self.P, self.V, self.tvals,
                                                exchange_grams=self._exchange, gather_curves=self._gather,
                                                timings=timings, block_ready=ready)
        bad = self.engine.check_numerics(self.lams)
        if bad is not None:
            f, j = bad
            raise SingularInterpolant(f"interpolated factor is singular at lambda={self.grid[j]} (fold {f})")
        return curves.cpu().numpy(), best.cpu().numpy()


_SESSION_CACHE = {}  # shape key -> CvSession (the most recent shape only)


def _cached_session(counts, d, m, grid_values, g, r, metric, holdout, raw_monomials):
    """A CvSession for these shapes and this grid, reused across drop-in calls.

    A session preallocates every device buffer of the sweep (about 18 GB at c4), so repeated
    grid_search_pichol calls on the same shapes -- the reference's usage pattern: one call per
    target or per dataset of a fixed design -- allocate once. Only the most recent shape is kept,
    so switching shapes releases the previous buffers."""
    import torch

    key = (tuple(int(c) for c in counts), int(d), int(m), np.asarray(grid_values, dtype=float).tobytes(), int(g),
           int(r), metric, holdout, bool(raw_monomials),
           torch.cuda.current_device() if torch.cuda.is_available() else -1)
    sess = _SESSION_CACHE.get(key)
    if sess is None:
        _SESSION_CACHE.clear()
        sess = CvSession(counts, d, m, grid_values, g=g, r=r, metric=metric, holdout=holdout,
                         raw_monomials=raw_monomials)
        _SESSION_CACHE[key] = sess
    return sess


def clear_session_cache():
    """Release the device buffers held for repeated grid_search_pichol calls."""
    _SESSION_CACHE.clear()


def grid_search_pichol(
    p,
    grid,
    folds,
    metric=RMSE,
    g=4,
    r=2,
    layout_kind=trivec.RECURSIVE,
    h0=64,
    raw_monomials=False,
    threads=None,
    holdout="auto",
):
    """Fit the factor polynomials per fold, then sweep the grid on the device (cvsearch.py:206-243).

    ``layout_kind``/``h0`` are validated for compatibility; the device always packs
    factors in the tile layout, which gives the same fitted values (the fit is
    per entry, so it is layout independent, tests/test_pichol.py:73-83).
    """
    if g > grid.q:
        raise UsageError(f"cannot draw g={g} samples from a grid of {grid.q}")
    if metric not in METRICS:
        raise UsageError(f"unknown metric {metric!r}")
    threads = resolve_threads(threads)
    t_start = time.perf_counter()
    if layout_kind not in trivec.ALL_KINDS:
        raise DimensionMismatch(f"unknown layout kind {layout_kind!r}")
    if layout_kind == trivec.RECURSIVE and h0 < 1:
        raise InvalidThreshold(f"recursion threshold must be >= 1, got {h0}")
    X, Y, counts = prepare_design(p, folds)
    n, d = X.shape
    sess = _cached_session(counts, d, Y.shape[1], grid.values, g, r, metric, holdout, raw_monomials)
    timings = {}
    curves, _ = sess.run(X, Y, timings=timings)
    k = folds.k
    per_fold = _zero_timings()
    per_fold["factorize"] = timings.get("factorize", 0.0) / k
    per_fold["fit"] = timings.get("fit", 0.0) / k
    per_fold["interp"] = timings.get("interp", 0.0) / k
    per_fold["predict"] = (timings.get("predict_local", 0.0) + timings.get("predict", 0.0)) / k
    return _merge("pichol", grid.values, curves, per_fold, time.perf_counter() - t_start)


def grid_search_exact(p, grid, folds, metric=RMSE, threads=None, holdout="auto"):
    """One exact factorization per fold per grid point, on the device (cvsearch.py:178-203).

    The paper's Chol baseline: H_f + lam I is factored for every lam (batches of 32 per
    rp_potrf_batched call) and solved with the same fused substitution kernel, q = 1."""
    from . import exact

    if metric not in METRICS:
        raise UsageError(f"unknown metric {metric!r}")
    threads = resolve_threads(threads)
    t_start = time.perf_counter()
    X, Y, counts = prepare_design(p, folds)
    curves = exact.exact_curves(X, Y, counts, grid.values, metric=metric, holdout=holdout)
    wall = time.perf_counter() - t_start
    per_fold = _zero_timings()
    per_fold["factorize"] = wall / folds.k
    return _merge("chol", grid.values, curves, per_fold, wall)


def mchol_search(p, c0, s0_init, s_min, folds, metric=RMSE, threads=None, holdout="auto"):
    """Three-point log-scale narrowing with exact solves (cvsearch.py:246-320), on the device.

    Each round evaluates the new candidates of {c - s, c, c + s} (log10 lambda) for all folds in
    one batched factorization; the fold-mean error (and, for several outputs, its mean over the
    outputs) picks the next center; s halves until s <= s_min. Per fold the factorization count
    is exactly 3 + 2 * ceil(log2(s0_init / s_min)), as in the reference."""
    from . import exact

    if not s0_init > s_min > 0:
        raise UsageError(f"need s0_init > s_min > 0, got {s0_init}, {s_min}")
    if metric not in METRICS:
        raise UsageError(f"unknown metric {metric!r}")
    threads = resolve_threads(threads)
    t_start = time.perf_counter()
    X, Y, counts = prepare_design(p, folds)
    ev = exact.ExactEvaluator(X, Y, counts, metric=metric, holdout=holdout)
    cache = {}

    def evaluate(lcs):
        new = [lc for lc in dict.fromkeys(lcs) if lc not in cache]
        if new:
            curves = ev.eval(np.array([10.0 ** lc for lc in new]))  # (k, len(new), m)
            fold_mean = np.mean(curves, axis=0)  # fold-ordered mean (cvsearch.py:290)
            for j, lc in enumerate(new):
                e = fold_mean[j]
                cache[lc] = float(e[0]) if e.shape[0] == 1 else float(np.mean(e))
        return [cache[lc] for lc in lcs]

    c, s = float(c0), float(s0_init)
    while True:
        cands = [c - s, c, c + s]
        vals = evaluate(cands)
        c = cands[int(np.argmin(vals))]
        if s <= s_min:
            break
        s /= 2.0
    wall = time.perf_counter() - t_start
    evaluated = sorted(cache)
    lams = np.array([10.0 ** lc for lc in evaluated])
    errs = np.array([cache[lc] for lc in evaluated])
    rows = [{"fold": -1, "lambda": float(l), "error": float(e), **_zero_timings()} for l, e in zip(lams, errs)]
    timings = _zero_timings()
    timings["factorize"] = wall
    best_idx = int(np.argmin(errs))
    return CvReport(
        method="mchol",
        per_lambda_error={float(l): float(e) for l, e in zip(lams, errs)},
        best_lambda=float(lams[best_idx]),
        best_error=float(errs[best_idx]),
        timings=timings,
        rows=rows,
        wall_seconds=wall,
    )


def pinrmse_search(p, grid, folds, metric=RMSE, g=4, r=2, threads=None, holdout="auto"):
    """Interpolate the hold-out error curve itself from g exact points (cvsearch.py:322-380).

    The g sampled exact errors (device, all folds in one batch) are averaged over folds; the
    degree-r polynomial fit and its minimizer over the grid are the reference's host
    arithmetic on those g numbers (same V, same COND_LIMIT rescale, same Cholesky of V^T V)."""
    import scipy.linalg

    from . import exact

    if g <= r:
        raise UsageError(f"need more samples than the degree: g={g}, r={r}")
    if g > grid.q:
        raise UsageError(f"cannot draw g={g} samples from a grid of {grid.q}")
    if metric not in METRICS:
        raise UsageError(f"unknown metric {metric!r}")
    threads = resolve_threads(threads)
    t_start = time.perf_counter()
    sample_lams = grid.values[pichol.sample_indices(grid.q, g)]
    X, Y, counts = prepare_design(p, folds)
    ev = exact.ExactEvaluator(X, Y, counts, metric=metric, holdout=holdout)
    curves = ev.eval(sample_lams)  # (k, g, m)
    fold_errs = curves[:, :, 0] if curves.shape[2] == 1 else np.mean(curves, axis=2)
    mean_errs = np.mean(fold_errs, axis=0)
    lams = np.asarray(sample_lams, dtype=float)
    V = np.vander(lams, r + 1, increasing=True)
    t_scale, t_shift = 1.0, 0.0
    if float(np.linalg.cond(V)) > pichol.COND_LIMIT:
        span = lams[-1] - lams[0]
        t_scale = 2.0 / span
        t_shift = -(lams[-1] + lams[0]) / span
        V = np.vander(t_scale * lams + t_shift, r + 1, increasing=True)
    Lv = scipy.linalg.cholesky(V.T @ V, lower=True, check_finite=False)
    w = scipy.linalg.solve_triangular(Lv, V.T @ mean_errs, lower=True, check_finite=False)
    coeff = scipy.linalg.solve_triangular(Lv.T, w, lower=False, check_finite=False)
    fitted = np.vander(t_scale * grid.values + t_shift, r + 1, increasing=True) @ coeff
    wall = time.perf_counter() - t_start
    per_fold = _zero_timings()
    per_fold["factorize"] = wall / folds.k
    rows = []
    for i in range(folds.k):
        for lam, e in zip(sample_lams, fold_errs[i]):
            rows.append({"fold": i, "lambda": float(lam), "error": float(e), **per_fold})
    for lam, e in zip(grid.values, fitted):
        rows.append({"fold": -1, "lambda": float(lam), "error": float(e), **_zero_timings()})
    timings = _zero_timings()
    timings["factorize"] = wall
    best_idx = int(np.argmin(fitted))
    return CvReport(
        method="pinrmse",
        per_lambda_error={float(l): float(e) for l, e in zip(grid.values, fitted)},
        best_lambda=float(grid.values[best_idx]),
        best_error=float(fitted[best_idx]),
        timings=timings,
        rows=rows,
        wall_seconds=wall,
        curves=curves,
    )


def _fit_basis_checked(sample_lams, r, raw_monomials):
    from .errors import DegenerateSamples, InsufficientSamples

    lams = np.asarray(sample_lams, dtype=float)
    if lams.shape[0] <= r:
        raise InsufficientSamples(f"need more samples than the degree: g={lams.shape[0]}, r={r}")
    if np.unique(lams).shape[0] != lams.shape[0]:
        raise DegenerateSamples("sample lambdas must be distinct")
    if np.any(lams <= 0):
        raise DegenerateSamples("sample lambdas must be positive")
    return pichol.fit_basis(lams, r, raw_monomials)


CSV_HEADER = "method,fold,lambda,error," + ",".join(f"t_{ph}" for ph in PHASES)


def report_csv_lines(report):
    """Render a CvReport as CSV lines, header first (cvsearch.py:429-444)."""
    lines = [CSV_HEADER]
    for row in report.rows:
        cells = [report.method, str(row["fold"]), f"{row['lambda']:.17g}", f"{row['error']:.17g}"]
        cells += [f"{row[ph]:.6g}" for ph in PHASES]
        lines.append(",".join(cells))
    return lines
