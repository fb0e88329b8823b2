"""Exact-Cholesky cross-validation on the device (SURVEY.md 8(f) "next" row 1).

``grid_search_exact`` (cvsearch.py:178-203) factors H_f + lambda I at every grid point of
every fold. On the B200 it reuses the piCholesky kernels without interpolation:

  rp_gram_blocks / rp_fold_systems   H_f = sum_b G_b - G_f, rhs_f, shifted by a batch of lambdas
  rp_potrf_batched                   up to 32 exact factors at once
  rp_fit_tiles (s = 1, degree 0)     each factor packed into the tile layout as its own "model"
  rp_eval_solve (q = 1)              fused blocked forward/back substitution per factor
  rp_holdout_gram / _direct          hold-out errors

It is the paper's Chol baseline (Table 2) on the same hardware and a device-side
exact reference for the interpolated sweep.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _lib
from ._lib import call, ptr, stream
from .engine import MAX_M_PER_SOLVE, MISCLASS, RMSE, padded, tile_elems
from .errors import NotPositiveDefinite, UsageError

MAX_BATCH = 32  # rp_fold_systems handles up to 32 shifts per call


def exact_curves(X, Y, block_rows, grid, metric=RMSE, holdout="auto", batch=MAX_BATCH):
    """Per-fold exact hold-out curves (k, q, m) for rows grouped by fold (block b = fold b)."""
    torch = _dev.torch()
    _lib.require_cuda()
    X = np.ascontiguousarray(X, dtype=np.float64)
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    n, d = X.shape
    m = Y.shape[1]
    k = len(block_rows)
    grid = np.asarray(grid, dtype=np.float64)
    q = grid.shape[0]
    if holdout == "auto":
        holdout = "gram" if metric == RMSE else "direct"
    if holdout == "gram" and metric != RMSE:
        raise UsageError("the Gram-form hold-out error supports RMSE only")
    metric_id = _lib.RP_METRIC_RMSE if metric == RMSE else _lib.RP_METRIC_MISCLASS
    row_off = np.concatenate([[0], np.cumsum(block_rows)]).astype(np.int64)
    dp = padded(d)
    st = stream()
    dX, dY = _dev.to_dev(X), _dev.to_dev(Y)
    G = _dev.empty((k, d, d))
    C = _dev.empty((k, m, d))
    yy = _dev.empty((k, m))
    ws_gram = _dev.workspace(_lib.query("rp_gram_workspace_size", d, int(max(block_rows)), 1))
    for b in range(k):
        off, rows = int(row_off[b]), int(block_rows[b])
        call("rp_gram_blocks", ptr(dX[off:]), d, rows, 1, d, ptr(dY[off:]), m, m, ptr(G[b]), ptr(C[b]), ptr(ws_gram),
             st)
        call("rp_col_sumsq", ptr(dY[off:]), m, rows, 1, m, ptr(yy[b]), st)
    B = max(1, min(batch, MAX_BATCH, q))
    Gsum = _dev.empty((d, d))
    A = _dev.empty((B, d, d))
    rhs = _dev.empty((1, dp, m))
    theta = _dev.empty((B, tile_elems(d, 1)))
    resid = _dev.empty((B,))
    info = _dev.zeros((B,), dtype=torch.int32)
    ws_potrf = _dev.workspace(_lib.query("rp_potrf_workspace_size", d, B))
    ws_fit = _dev.workspace(_lib.query("rp_fit_workspace_size", d, B))
    one = np.ones((1, 1))
    zero_t = _dev.zeros((1,))
    groups = [(c, min(c + MAX_M_PER_SOLVE, m)) for c in range(0, m, MAX_M_PER_SOLVE)]
    curves = np.empty((k, q, m))
    for f in range(k):
        if holdout == "gram":
            call("rp_symmetrize", ptr(G[f]), d, d * d, 1, st)
        n_val = int(block_rows[f])
        for j0 in range(0, q, B):
            lams = np.ascontiguousarray(grid[j0:j0 + B])
            nb = lams.shape[0]
            folds = np.array([f], dtype=np.int32)
            call("rp_fold_systems", ptr(G), ptr(C), k, d, m, _lib.host_ptr(folds), 1, _lib.host_ptr(lams), nb,
                 ptr(Gsum), ptr(A), ptr(rhs), st)
            call("rp_potrf_batched", ptr(A), d, d * d, nb, ptr(info), ptr(ws_potrf), st)
            bad = info[:nb].cpu().numpy()
            if np.any(bad != 0):
                i = int(np.flatnonzero(bad)[0])
                raise NotPositiveDefinite(
                    f"leading minor of order {int(bad[i])} is not positive definite (fold {f}, lambda={lams[i]})")
            call("rp_fit_tiles", ptr(A), d, 1, nb, 0, _lib.host_ptr(one), _lib.host_ptr(one), ptr(theta), ptr(resid),
                 ptr(ws_fit), st)
            for c0, c1 in groups:
                mg = c1 - c0
                rhs_b = rhs[:, :, c0:c1].expand(nb, dp, mg).contiguous()
                ldw = mg + (mg & 1)
                W = _dev.empty((nb, dp, ldw))
                flags = _dev.zeros((nb,), dtype=torch.int32)
                ws = _dev.workspace(_lib.query("rp_eval_solve_workspace_size", d, 0, nb, mg, 1))
                call("rp_eval_solve", ptr(theta), d, 0, nb, ptr(rhs_b), mg, ptr(zero_t), 1, ptr(W), ldw, ptr(flags),
                     ptr(ws), st)
                out = _dev.empty((nb, 1, mg))
                if holdout == "gram":
                    yy_b = yy[f, c0:c1].expand(nb, mg).contiguous()
                    wsh = _dev.workspace(_lib.query("rp_holdout_workspace_size", n_val, d, 1, mg, nb))
                    call("rp_holdout_gram", ptr(G[f]), 0, ptr(C[f, c0:]), 0, ptr(yy_b), n_val, d, mg, ptr(W), ldw,
                         dp * ldw, 1, nb, ptr(out), ptr(wsh), st)
                else:
                    off = int(row_off[f])
                    wsh = _dev.workspace(_lib.query("rp_holdout_workspace_size", n_val, d, 1, mg, nb))
                    call("rp_holdout_direct", ptr(dX[off:]), d, 0, n_val, d, ptr(dY[off:, c0:]), m, mg, ptr(W), ldw,
                         dp * ldw, 1, nb, metric_id, ptr(out), ptr(wsh), st)
                curves[f, j0:j0 + nb, c0:c1] = out[:, 0, :].cpu().numpy()
    return curves
