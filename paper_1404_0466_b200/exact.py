"""Exact-Cholesky hold-out errors on the device (SURVEY.md 8(f) "next" rows 1 and 4).

``grid_search_exact`` (cvsearch.py:178-203), ``mchol_search`` (cvsearch.py:246-320) and
``pinrmse_search`` (cvsearch.py:322-380) all need the hold-out error of the exact solution at
arbitrary lambdas: factor H_f + lambda I, solve, score. ``ExactEvaluator`` keeps the fold
Gram blocks resident and evaluates any set of lambdas for all folds at once, reusing the
piCholesky kernels without interpolation:

  rp_gram_blocks / rp_fold_systems   H_f = sum_{b != f} G_b, rhs_f, shifted by each lambda
  rp_potrf_batched                   up to 32 exact factors per call (folds x lambdas)
  rp_fit_tiles (s = 1, degree 0)     each factor packed into the tile layout as its own "model"
  rp_eval_solve (q = 1)              fused blocked forward/back substitution per factor
  rp_holdout_gram / _direct          hold-out errors
"""

from __future__ import annotations

import numpy as np

from . import _dev, _lib
from ._lib import call, ptr, stream
from .engine import MAX_M_PER_SOLVE, RMSE, padded, tile_elems
from .errors import NotPositiveDefinite, UsageError

MAX_BATCH = 32  # matrices per rp_potrf_batched / rp_fold_systems call


class ExactEvaluator:
    """Per-fold exact hold-out errors for rows grouped by fold (block b = fold b)."""

    def __init__(self, X, Y, block_rows, metric=RMSE, holdout="auto"):
        torch = _dev.torch()
        _lib.require_cuda()
        X = np.ascontiguousarray(X, dtype=np.float64)
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        self.n, self.d = X.shape
        self.m = Y.shape[1]
        self.k = len(block_rows)
        self.block_rows = [int(b) for b in block_rows]
        if holdout == "auto":
            holdout = "gram" if metric == RMSE else "direct"
        if holdout == "gram" and metric != RMSE:
            raise UsageError("the Gram-form hold-out error supports RMSE only")
        self.holdout = holdout
        self.metric_id = _lib.RP_METRIC_RMSE if metric == RMSE else _lib.RP_METRIC_MISCLASS
        self.row_off = np.concatenate([[0], np.cumsum(self.block_rows)]).astype(np.int64)
        d, m, k = self.d, self.m, self.k
        self.dp = padded(d)
        st = stream()
        self.dX, self.dY = _dev.to_dev(X), _dev.to_dev(Y)
        self.G = _dev.empty((k, d, d))
        self.C = _dev.empty((k, m, d))
        self.yy = _dev.empty((k, m))
        ws_gram = _dev.workspace(_lib.query("rp_gram_workspace_size", d, max(self.block_rows), 1))
        for b in range(k):
            off, rows = int(self.row_off[b]), self.block_rows[b]
            call("rp_gram_blocks", ptr(self.dX[off:]), d, rows, 1, d, ptr(self.dY[off:]), m, m, ptr(self.G[b]),
                 ptr(self.C[b]), ptr(ws_gram), st)
            call("rp_col_sumsq", ptr(self.dY[off:]), m, rows, 1, m, ptr(self.yy[b]), st)
        self.groups = [(c, min(c + MAX_M_PER_SOLVE, m)) for c in range(0, m, MAX_M_PER_SOLVE)]
        self._torch = torch

    def eval(self, lams, folds=None):
        """Hold-out errors (len(folds), len(lams), m) of the exact solutions at `lams`."""
        lams = np.ascontiguousarray(lams, dtype=np.float64).reshape(-1)
        folds = list(range(self.k)) if folds is None else [int(f) for f in folds]
        nl = lams.shape[0]
        out = np.empty((len(folds), nl, self.m))
        lb = max(1, min(nl, MAX_BATCH))  # lambdas per call
        fb = max(1, MAX_BATCH // lb)      # folds per call
        for i0 in range(0, len(folds), fb):
            fs = folds[i0:i0 + fb]
            for j0 in range(0, nl, lb):
                out[i0:i0 + len(fs), j0:j0 + lb] = self._batch(fs, lams[j0:j0 + lb])
        return out

    def _batch(self, folds, lams):
        torch = self._torch
        d, m, dp, k = self.d, self.m, self.dp, self.k
        nf, nb = len(folds), lams.shape[0]
        nmod = nf * nb  # models in fold-major order: f * nb + j
        st = stream()
        A = _dev.empty((nmod, d, d))
        rhs = _dev.empty((nf, dp, m))
        fa = np.ascontiguousarray(folds, dtype=np.int32)
        call("rp_fold_systems", ptr(self.G), ptr(self.C), k, d, m, _lib.host_ptr(fa), nf, _lib.host_ptr(lams), nb,
             ptr(A), ptr(rhs), st)
        info = _dev.zeros((nmod,), dtype=torch.int32)
        ws = _dev.workspace(_lib.query("rp_potrf_workspace_size", d, nmod))
        call("rp_potrf_batched", ptr(A), d, d * d, nmod, ptr(info), ptr(ws), st)
        bad = info.cpu().numpy()
        if np.any(bad != 0):
            i = int(np.flatnonzero(bad)[0])
            raise NotPositiveDefinite(f"leading minor of order {int(bad[i])} is not positive definite "
                                      f"(fold {folds[i // nb]}, lambda={lams[i % nb]})")
        theta = _dev.empty((nmod, tile_elems(d, 1)))
        resid = _dev.empty((nmod,))
        one = np.ones((1, 1))
        call("rp_fit_tiles", ptr(A), d, 1, nmod, 0, _lib.host_ptr(one), _lib.host_ptr(one), ptr(theta), ptr(resid),
             ptr(_dev.workspace(_lib.query("rp_fit_workspace_size", d, nmod, 1, 0))), st)
        del A
        zero_t = _dev.zeros((1,))
        out = np.empty((nf, nb, m))
        for c0, c1 in self.groups:
            mg = c1 - c0
            rhs_b = rhs[:, :, c0:c1].unsqueeze(1).expand(nf, nb, dp, mg).reshape(nmod, dp, mg).contiguous()
            ldw = mg + (mg & 1)
            W = _dev.empty((nmod, dp, ldw))
            flags = _dev.zeros((nmod,), dtype=torch.int32)
            wss = _dev.workspace(_lib.query("rp_eval_solve_workspace_size", d, 0, nmod, mg, 1))
            call("rp_eval_solve", ptr(theta), d, 0, nmod, ptr(rhs_b), mg, ptr(zero_t), 1, ptr(W), ldw, ptr(flags),
                 ptr(wss), st)
            for i, f in enumerate(folds):
                n_val = self.block_rows[f]
                res = _dev.empty((nb, 1, mg))
                Wf = W[i * nb:(i + 1) * nb]
                wsh = _dev.workspace(_lib.query("rp_holdout_workspace_size", n_val, d, 1, mg, nb))
                if self.holdout == "gram":
                    yy_b = self.yy[f, c0:c1].expand(nb, mg).contiguous()
                    off = int(self.row_off[f])
                    call("rp_holdout_gram", ptr(self.G[f]), 0, ptr(self.C[f, c0:]), 0, ptr(yy_b), n_val, d, mg,
                         ptr(Wf), ldw, dp * ldw, 1, nb, ptr(self.dX[off:]), d, 0, ptr(self.dY[off:, c0:]), m,
                         ptr(res), ptr(wsh), st)
                else:
                    off = int(self.row_off[f])
                    call("rp_holdout_direct", ptr(self.dX[off:]), d, 0, n_val, d, ptr(self.dY[off:, c0:]), m, mg,
                         ptr(Wf), ldw, dp * ldw, 1, nb, self.metric_id, ptr(res), ptr(wsh), st)
                out[i, :, c0:c1] = res[:, 0, :].cpu().numpy()
        return out


def exact_curves(X, Y, block_rows, grid, metric=RMSE, holdout="auto", batch=MAX_BATCH):
    """Per-fold exact hold-out curves (k, q, m) over a grid (grid_search_exact)."""
    ev = ExactEvaluator(X, Y, block_rows, metric=metric, holdout=holdout)
    grid = np.asarray(grid, dtype=np.float64)
    out = np.empty((ev.k, grid.shape[0], ev.m))
    b = max(1, min(batch, MAX_BATCH))
    for j0 in range(0, grid.shape[0], b):
        out[:, j0:j0 + b] = ev.eval(grid[j0:j0 + b])
    return out
