"""Device pipeline of the piCholesky cross-validation sweep.

One ``PicholEngine`` owns every device buffer of a sweep (allocated once, reused
across calls -- no allocation on the hot path) and launches the six stages of
SURVEY.md 8(a) through the C ABI on the current torch CUDA stream:

  (1) rp_gram_blocks      G_b = X_b^T X_b, C_b = X_b^T Y_b per fold block   ridge.py:50-60
      rp_fold_systems     A_{f,s} = sum_{b != f} G_b + lam_s I, rhs_f       pichol.py:105
  (2) rp_potrf_batched    L_{f,s} = chol(A_{f,s}) for all local folds x s   linalg.py:98
  (3+4) rp_fit_tiles      theta_f = P T_f in the tile layout + residual     pichol.py:109-125
  (5) rp_eval_solve       W_f(lam_j) for all q lambdas, fused eval+solve    ridge.py:78-91
  (6) rp_holdout_*        per (fold, lambda, output) hold-out error         cvsearch.py:106-123
      rp_select           fold mean + first argmin                          cvsearch.py:154-175

Folds are contiguous row blocks of the (fold-grouped) design: block b holds the
validation rows of fold b, so the training Hessian of fold f is
sum_{b != f} G_b. Multi-GPU sharding plugs in through the
``exchange_grams`` / ``gather_curves`` hooks (see ``dist.py``).
"""

from __future__ import annotations

import math
import time

import numpy as np

from . import _lib
from ._lib import call, ptr, stream
from .errors import NotPositiveDefinite, SingularInterpolant, UsageError

RMSE = "rmse"
MISCLASS = "misclass"

TILE = 64
MAX_M_PER_SOLVE = 16


def padded(d):
    return TILE * ((d + TILE - 1) // TILE)


def tile_elems(d, P):
    """Doubles of one fold's coefficient buffer (tile layout, include/ridgepath_b200.h)."""
    return int(_lib.query("rp_theta_size", d, P - 1))


def _resolve(block_ready, b):
    """The upload event of block b (starting a deferred upload first, see stage_gram)."""
    ev = block_ready[b]
    if callable(ev):
        ev = block_ready[b] = ev()
    return ev


class PicholEngine:
    """Preallocated device state for ``grid_search_pichol`` on one GPU.

    block_rows: rows of each fold block, in fold order (fold b = block b).
    local_folds: folds whose curves this device computes (default: all).
    gram_blocks: blocks whose Gram this device computes (default: all); the rest
        must be filled by ``exchange_grams``.
    """

    def __init__(self, block_rows, d, m, q, s, r, local_folds=None, gram_blocks=None, metric=RMSE,
                 holdout="auto", device=None):
        import torch

        _lib.require_cuda()
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        self.block_rows = [int(b) for b in block_rows]
        self.k = len(self.block_rows)
        if self.k < 1:
            raise UsageError("need at least one fold")
        self.row_off = np.concatenate([[0], np.cumsum(self.block_rows)]).astype(np.int64)
        self.n = int(self.row_off[-1])
        self.d, self.m, self.q, self.s, self.r = int(d), int(m), int(q), int(s), int(r)
        self.P = self.r + 1
        self.dp = padded(self.d)
        self.local_folds = list(range(self.k)) if local_folds is None else [int(f) for f in local_folds]
        self.gram_blocks = list(range(self.k)) if gram_blocks is None else [int(b) for b in gram_blocks]
        self.nf = len(self.local_folds)
        if metric not in (RMSE, MISCLASS):
            raise UsageError(f"unknown metric {metric!r}")
        self.metric = metric
        if holdout == "auto":
            holdout = "gram" if metric == RMSE else "direct"
        if holdout == "gram" and metric != RMSE:
            raise UsageError("the Gram-form hold-out error supports RMSE only")
        self.holdout = holdout
        self.equal_blocks = len(set(self.block_rows)) == 1
        # output groups for the fused solve (<= 16 outputs per launch)
        self.groups = [(c, min(c + MAX_M_PER_SOLVE, self.m)) for c in range(0, self.m, MAX_M_PER_SOLVE)]
        self._alloc()

    # ------------------------------------------------------------------ buffers
    def _alloc(self):
        torch, dev = self.torch, self.device
        f64 = dict(dtype=torch.float64, device=dev)
        d, dp, k, nf, s, q, m = self.d, self.dp, self.k, self.nf, self.s, self.q, self.m
        if nf == 0:  # a rank without folds (world > k): it only joins the curve exchange
            self.curves = torch.empty((0, q, m), **f64)
            self.mean = torch.empty((q, m), **f64)
            self.best = torch.empty((m,), dtype=torch.int32, device=dev)
            self.info = torch.zeros((0,), dtype=torch.int32, device=dev)
            self.flags = torch.zeros((len(self.groups), 0, q), dtype=torch.int32, device=dev)
            self.tvals = torch.empty((q,), **f64)
            return
        self.G = torch.empty((k, d, d), **f64)
        self.C = torch.empty((k, m, d), **f64)  # C_b column-major d x m == (m, d) row-major
        self.yy = torch.empty((k, m), **f64)
        self.A = torch.empty((nf, s, d, d), **f64)
        self.theta = torch.empty((nf, tile_elems(d, self.P)), **f64)
        self.resid = torch.empty((nf,), **f64)
        self.rhs = torch.empty((nf, dp, m), **f64)
        self.info = torch.zeros((nf * s,), dtype=torch.int32, device=dev)
        self.flags = torch.zeros((len(self.groups), nf, q), dtype=torch.int32, device=dev)
        self.W = []
        self.rhs_g = []
        for c0, c1 in self.groups:
            mg = c1 - c0
            ldw = q * mg + ((q * mg) & 1)
            self.W.append(torch.empty((nf, dp, ldw), **f64))
            self.rhs_g.append(self.rhs if len(self.groups) == 1 else torch.empty((nf, dp, mg), **f64))
        self.curves = torch.empty((nf, q, m), **f64)
        self.curves_g = [self.curves if len(self.groups) == 1 else torch.empty((nf, q, c1 - c0), **f64)
                         for c0, c1 in self.groups]
        self.mean = torch.empty((q, m), **f64)
        self.best = torch.empty((m,), dtype=torch.int32, device=dev)
        self.tvals = torch.empty((q,), **f64)
        u8 = dict(dtype=torch.uint8, device=dev)
        # tensor-core (Ozaki) Gram slices: sized for both call patterns of stage_gram
        ng = len(self.gram_blocks)
        self.ws_gram = torch.empty((max(_lib.query("rp_gram_workspace_size", d, self.block_rows[0], ng),
                                        _lib.query("rp_gram_workspace_size", d, max(self.block_rows), 1)),), **u8)
        self.ws_potrf = torch.empty((_lib.query("rp_potrf_workspace_size", d, nf * s),), **u8)
        self.ws_fit = torch.empty((_lib.query("rp_fit_workspace_size", d, nf, s, self.r),), **u8)
        nval = max(self.block_rows[f] for f in self.local_folds)
        mg = max(c1 - c0 for c0, c1 in self.groups)
        self.ws_hold = torch.empty((_lib.query("rp_holdout_workspace_size", nval, d, q, mg, 1 if not self.equal_blocks else nf),), **u8)
        self.ws_solve = torch.empty((max(_lib.query("rp_eval_solve_workspace_size", d, self.r, n, c1 - c0, q)
                                         for c0, c1 in self.groups for n in {max(nf - 1, 1), nf}),), **u8)

    def device_bytes(self):
        tot = 0
        for name, v in vars(self).items():
            if hasattr(v, "element_size") and hasattr(v, "numel"):
                tot += v.element_size() * v.numel()
            elif isinstance(v, list):
                tot += sum(t.element_size() * t.numel() for t in v if hasattr(t, "numel"))
        return tot

    # ------------------------------------------------------------------ stages
    def stage_gram(self, X, Y, block_ready=None, blocks=None):
        """Gram blocks. block_ready: optional {block: cuda.Event} -- the Gram of a block then waits
        only for that block's upload, so the host->device copy of later blocks overlaps it. A value
        may also be a callable that starts the block's upload and returns its event; it is called
        (and replaced by the event) right before that block's Gram is enqueued.
        blocks: a subset of this engine's Gram blocks (default all)."""
        d, m = self.d, self.m
        st = stream()
        blocks = self.gram_blocks if blocks is None else blocks
        contiguous = blocks == list(range(blocks[0], blocks[0] + len(blocks)))
        if self.equal_blocks and contiguous and block_ready is None:
            b0 = blocks[0]
            rows = self.block_rows[0]
            off = int(self.row_off[b0])
            call("rp_gram_blocks", ptr(X[off:]), d, rows, len(blocks), d, ptr(Y[off:]), m, m,
                 ptr(self.G[b0]), ptr(self.C[b0]), ptr(self.ws_gram), st)
            if self.holdout == "gram":
                call("rp_col_sumsq", ptr(Y[off:]), m, rows, len(blocks), m, ptr(self.yy[b0]), st)
        else:
            cur = self.torch.cuda.current_stream()
            for b in blocks:
                if block_ready is not None:
                    cur.wait_event(_resolve(block_ready, b))
                off, rows = int(self.row_off[b]), self.block_rows[b]
                call("rp_gram_blocks", ptr(X[off:]), d, rows, 1, d, ptr(Y[off:]), m, m,
                     ptr(self.G[b]), ptr(self.C[b]), ptr(self.ws_gram), st)
                if self.holdout == "gram":
                    call("rp_col_sumsq", ptr(Y[off:]), m, rows, 1, m, ptr(self.yy[b]), st)

    def stage_systems(self, sample_lams, part=None, nblocks=None):
        """Shifted systems of the local folds part = (i0, i1): A_{f,s} = sum_{b != f} G_b + lam_s I.
        nblocks: sum only the first nblocks Gram blocks (a fold whose own block is not among them
        gets the same, bit-identical sum as with all blocks)."""
        i0, i1 = part if part is not None else (0, self.nf)
        folds = np.ascontiguousarray(self.local_folds[i0:i1], dtype=np.int32)
        lams = np.ascontiguousarray(sample_lams, dtype=np.float64)
        nb = self.k if nblocks is None else nblocks
        call("rp_fold_systems", ptr(self.G), ptr(self.C), nb, self.d, self.m, _lib.host_ptr(folds), i1 - i0,
             _lib.host_ptr(lams), self.s, ptr(self.A[i0]), ptr(self.rhs[i0]), stream())

    def stage_factorize(self, part=None, ws=None):
        i0, i1 = part if part is not None else (0, self.nf)
        d = self.d
        call("rp_potrf_batched", ptr(self.A[i0]), d, d * d, (i1 - i0) * self.s, ptr(self.info[i0 * self.s:]),
             ptr(self.ws_potrf if ws is None else ws), stream())

    def stage_fit(self, Pmat, Vmat, part=None, ws=None):
        i0, i1 = part if part is not None else (0, self.nf)
        Pm = np.ascontiguousarray(Pmat, dtype=np.float64)
        Vm = np.ascontiguousarray(Vmat, dtype=np.float64)
        call("rp_fit_tiles", ptr(self.A[i0]), self.d, self.s, i1 - i0, self.r, _lib.host_ptr(Pm), _lib.host_ptr(Vm),
             ptr(self.theta[i0]), ptr(self.resid[i0:]), ptr(self.ws_fit if ws is None else ws), stream())

    def _solve_workspace(self):
        """The solve workspace for the current plan (rp_set_option("solve_lam" / "solve_cluster") may change
        the chunking after allocation: grow the buffer then instead of overrunning it)."""
        need = max(_lib.query("rp_eval_solve_workspace_size", self.d, self.r, n, c1 - c0, self.q)
                   for c0, c1 in self.groups for n in {max(self.nf - 1, 1), self.nf})
        if need > self.ws_solve.numel():
            self.ws_solve = self.torch.empty((need,), dtype=self.torch.uint8, device=self.device)
        return self.ws_solve

    def stage_solve(self, part=None, ws=None):
        i0, i1 = part if part is not None else (0, self.nf)
        if ws is None:
            ws = self._solve_workspace()
        for gi, (c0, c1) in enumerate(self.groups):
            if len(self.groups) > 1:
                self.rhs_g[gi][i0:i1].copy_(self.rhs[i0:i1, :, c0:c1])
            W = self.W[gi]
            call("rp_eval_solve", ptr(self.theta[i0]), self.d, self.r, i1 - i0, ptr(self.rhs_g[gi][i0]), c1 - c0,
                 ptr(self.tvals), self.q, ptr(W[i0]), W.shape[2], ptr(self.flags[gi][i0:]), ptr(ws), stream())

    def stage_holdout(self, X, Y):
        st = stream()
        metric = _lib.RP_METRIC_RMSE if self.metric == RMSE else _lib.RP_METRIC_MISCLASS
        d, q = self.d, self.q
        for gi, (c0, c1) in enumerate(self.groups):
            mg = c1 - c0
            W = self.W[gi]
            ldw = W.shape[2]
            out = self.curves_g[gi]
            if self.holdout == "gram":
                if self._folds_regular():
                    f0 = self.local_folds[0]
                    yyg = self.yy[:, c0:c1].contiguous() if len(self.groups) > 1 else self.yy
                    off = int(self.row_off[f0])
                    call("rp_holdout_gram", ptr(self.G[f0]), d * d, ptr(self.C[f0, c0:]), self.m * d,
                         ptr(yyg[f0]), self.block_rows[f0], d, mg, ptr(W), ldw, W[0].numel(), q, self.nf,
                         ptr(X[off:]), d, self.block_rows[0], ptr(Y[off:, c0:]), self.m,
                         ptr(out), ptr(self.ws_hold), st)
                else:
                    yyg = self.yy[:, c0:c1].contiguous()
                    for i, f in enumerate(self.local_folds):
                        off = int(self.row_off[f])
                        call("rp_holdout_gram", ptr(self.G[f]), d * d, ptr(self.C[f, c0:]), self.m * d,
                             ptr(yyg[f]), self.block_rows[f], d, mg, ptr(W[i]), ldw, W[0].numel(), q, 1,
                             ptr(X[off:]), d, 0, ptr(Y[off:, c0:]), self.m,
                             ptr(out[i]), ptr(self.ws_hold), st)
            else:
                if self._folds_regular():
                    f0 = self.local_folds[0]
                    off = int(self.row_off[f0])
                    call("rp_holdout_direct", ptr(X[off:]), d, self.block_rows[0], self.block_rows[0], d,
                         ptr(Y[off:, c0:]), self.m, mg, ptr(W), ldw, W[0].numel(), q, self.nf, metric, ptr(out),
                         ptr(self.ws_hold), st)
                else:
                    for i, f in enumerate(self.local_folds):
                        off = int(self.row_off[f])
                        call("rp_holdout_direct", ptr(X[off:]), d, self.block_rows[f], self.block_rows[f], d,
                             ptr(Y[off:, c0:]), self.m, mg, ptr(W[i]), ldw, W[0].numel(), q, 1, metric,
                             ptr(out[i]), ptr(self.ws_hold), st)
            if len(self.groups) > 1:
                self.curves[:, :, c0:c1].copy_(out)

    def _folds_regular(self):
        lf = self.local_folds
        return self.equal_blocks and lf == list(range(lf[0], lf[0] + len(lf)))

    def stage_select(self, curves_all):
        call("rp_select", ptr(curves_all), self.k, self.q, self.m, ptr(self.mean), ptr(self.best), stream())

    # ------------------------------------------------------------------ sweep
    def sweep(self, X, Y, sample_lams, Pmat, Vmat, tvals, exchange_grams=None, gather_curves=None,
              timings=None, block_ready=None):
        """Run stages (1)-(6). X: (n, d), Y: (n, m) float64 CUDA, rows grouped by fold block.
        tvals: (q,) host or device t values. Returns (curves_all, mean, best) device tensors."""
        torch = self.torch
        if isinstance(tvals, torch.Tensor):
            self.tvals.copy_(tvals, non_blocking=True)
        else:
            self.tvals.copy_(torch.from_numpy(np.ascontiguousarray(tvals, dtype=np.float64)), non_blocking=False)
        ev = [] if timings is not None else None

        def mark(name):
            if ev is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev.append((name, e))

        mark("start")
        if self.nf == 0:
            curves_all = gather_curves(self.curves) if gather_curves is not None else self.curves
            if curves_all.shape[0] == self.k:
                self.stage_select(curves_all)
                return curves_all, self.mean, self.best
            return curves_all, None, None
        self.stage_gram(X, Y, block_ready)
        if block_ready is not None:  # later stages may read any row of X / Y
            for b in list(block_ready):
                torch.cuda.current_stream().wait_event(_resolve(block_ready, b))
        if exchange_grams is not None:
            exchange_grams(self)
        self.stage_systems(sample_lams)
        mark("assemble")
        self.stage_factorize()
        mark("factorize")
        self.stage_fit(Pmat, Vmat)
        mark("fit")
        self.stage_solve()
        mark("interp")
        self.stage_holdout(X, Y)
        mark("predict_local")
        curves_all = gather_curves(self.curves) if gather_curves is not None else self.curves
        # the fold mean needs every fold's curve: a device holding only some folds and no gather
        # hook returns its local curves without a selection
        complete = curves_all.shape[0] == self.k
        if complete:
            self.stage_select(curves_all)
        mark("predict")
        if ev is not None:
            torch.cuda.synchronize()
            for (n0, e0), (n1, e1) in zip(ev[:-1], ev[1:]):
                timings[n1] = timings.get(n1, 0.0) + e0.elapsed_time(e1) / 1e3
        return (curves_all, self.mean, self.best) if complete else (curves_all, None, None)

    def check_numerics(self, sample_lams, info=None, flags=None):
        """Raise the reference's exceptions for device-side failures (host sync). info / flags: host copies
        taken earlier (a pipelined caller reads them back asynchronously), default the device buffers."""
        info = self.info.cpu().numpy() if info is None else info
        if np.any(info != 0):
            i = int(np.flatnonzero(info)[0])
            f, s = divmod(i, self.s)
            raise NotPositiveDefinite(
                f"leading minor of order {int(info[i])} is not positive definite "
                f"(fold {self.local_folds[f]}, lambda={float(sample_lams[s])})"
            )
        flags = self.flags.amax(dim=0).cpu().numpy() if flags is None else flags
        if np.any(flags != 0):
            f, j = np.argwhere(flags != 0)[0]
            return int(self.local_folds[f]), int(j)
        return None


def sweep_flops(k, n, d, m, q, s, r, nf=None, holdout="gram", n_val=None):
    """Algorithmic FP64 flop counts of one sweep, per stage."""
    nf = k if nf is None else nf
    n_val = n // k if n_val is None else n_val
    D = d * (d + 1) // 2
    out = {
        "gram": n * d * (d + 1) + 2.0 * n * d * m,
        "factorize": nf * s * d ** 3 / 3.0,
        "fit": 2.0 * nf * (r + 1) * s * D,
        "solve": nf * q * (2 * r + 4 * m) * D,
    }
    if holdout == "gram":
        # w^T G_f w from the lower triangle of the symmetric G_f: 2 * D flops per column
        out["holdout"] = nf * 2.0 * D * q * m
    else:
        out["holdout"] = nf * 2.0 * n_val * d * q * m
    return out


def solve_bytes(nf, d, r):
    """Algorithmic HBM bytes of the fused eval+solve: theta read once per pass (fwd + bwd)."""
    D = d * (d + 1) // 2
    return nf * 2 * (r + 1) * D * 8


def timed(fn):
    t0 = time.perf_counter()
    out = fn()
    return out, time.perf_counter() - t0


__all__ = ["PicholEngine", "sweep_flops", "solve_bytes", "padded", "tile_elems", "RMSE", "MISCLASS", "math"]
