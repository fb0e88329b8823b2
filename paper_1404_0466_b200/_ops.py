"""Single-problem device operations behind the drop-in API.

Thin wrappers that allocate per call (the API edge is not the hot path; the
sweep uses the preallocated ``engine.PicholEngine``) and launch the same C-ABI
kernels the sweep uses.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _lib
from ._lib import call, ptr, stream
from .engine import MAX_M_PER_SOLVE, padded, tile_elems


def gram(X, Y=None):
    """X^T X (full, exactly symmetric) and X^T Y on the device. X: (n, d) host."""
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    dX = _dev.to_dev(X)
    if Y is not None:
        Y2 = np.asarray(Y, dtype=np.float64).reshape(n, -1)
        m = Y2.shape[1]
        dY = _dev.to_dev(Y2)
    else:
        m, dY = 0, None
    G = _dev.empty((d, d))
    C = _dev.empty((max(m, 1), d))
    ws = _dev.workspace(_lib.query("rp_gram_workspace_size", d, n, 1))
    call("rp_gram_blocks", ptr(dX), d, n, 1, d, ptr(dY), max(m, 1), m, ptr(G), ptr(C) if m else None, ptr(ws),
         stream())
    call("rp_symmetrize", ptr(G), d, d * d, 1, stream())
    return G, (C[:m] if m else None)


def potrf(A_dev, d, batch):
    """In-place batched Cholesky of `batch` column-major d x d device matrices; returns info (host)."""
    info = _dev.zeros((batch,), dtype=_dev.torch().int32)
    ws = _dev.workspace(_lib.query("rp_potrf_workspace_size", d, batch))
    call("rp_potrf_batched", ptr(A_dev), d, d * d, batch, ptr(info), ptr(ws), stream())
    return info.cpu().numpy()


def lower_of(A_dev, d):
    """Zero the strict upper triangle of a column-major d x d device matrix (in place)."""
    t = _dev.torch()
    V = A_dev.view(d, d)  # V[j][i] = A(i, j)
    V.copy_(t.triu(V))
    return A_dev


def fit_tiles(L_dev, d, s, nf, r, Pmat, Vmat):
    """Tile-layout coefficients theta = P T of nf x s column-major factors; returns (theta, resid)."""
    P = r + 1
    theta = _dev.empty((nf, tile_elems(d, P)))
    resid = _dev.empty((nf,))
    ws = _dev.workspace(_lib.query("rp_fit_workspace_size", d, nf, s, r))
    Pm = np.ascontiguousarray(Pmat, dtype=np.float64)
    Vm = np.ascontiguousarray(Vmat, dtype=np.float64)
    call("rp_fit_tiles", ptr(L_dev), d, s, nf, r, _lib.host_ptr(Pm), _lib.host_ptr(Vm), ptr(theta), ptr(resid),
         ptr(ws), stream())
    return theta, resid


def pack_lower(L_dev, d):
    """Dense column-major lower factor -> tile layout with one plane (r = 0)."""
    theta, _ = fit_tiles(L_dev, d, 1, 1, 0, np.ones((1, 1)), np.ones((1, 1)))
    return theta


def eval_solve(theta_dev, d, r, rhs, tvals):
    """Solve L(t) L(t)^T W = rhs for each t in tvals with one fold's tile-layout theta.

    rhs: (d, m) host array. Returns (W (q, d, m) host, singular flags (q,) host)."""
    torch = _dev.torch()
    rhs = np.asarray(rhs, dtype=np.float64).reshape(d, -1)
    m = rhs.shape[1]
    tv = np.ascontiguousarray(np.atleast_1d(tvals), dtype=np.float64)
    q = tv.shape[0]
    dp = padded(d)
    dt = _dev.to_dev(tv)
    out = np.empty((q, d, m))
    flags = np.zeros(q, dtype=np.int32)
    for c0 in range(0, m, MAX_M_PER_SOLVE):
        c1 = min(c0 + MAX_M_PER_SOLVE, m)
        mg = c1 - c0
        R = _dev.zeros((dp, mg))
        R[:d].copy_(torch.from_numpy(np.ascontiguousarray(rhs[:, c0:c1])))
        ldw = q * mg + ((q * mg) & 1)
        W = _dev.empty((dp, ldw))
        fl = _dev.zeros((q,), dtype=torch.int32)
        ws = _dev.workspace(_lib.query("rp_eval_solve_workspace_size", d, r, 1, mg, q))
        call("rp_eval_solve", ptr(theta_dev), d, r, 1, ptr(R), mg, ptr(dt), q, ptr(W), ldw, ptr(fl), ptr(ws),
             stream())
        Wh = W[:d, : q * mg].cpu().numpy().reshape(d, q, mg)
        out[:, :, c0:c1] = np.transpose(Wh, (1, 0, 2))
        flags |= fl.cpu().numpy()
    return out, flags


def materialize(theta_dev, d, r, t):
    """Dense F-ordered L(t) from one fold's tile-layout theta (pichol.eval arithmetic)."""
    L = _dev.empty((d * d,))
    call("rp_eval_materialize", ptr(theta_dev), d, r, float(t), ptr(L), stream())
    return _dev.colmajor_to_host(L, d)


def export_theta(theta_dev, d, r, perm, D):
    """(r+1, D) coefficients in a reference VecLayout order (perm None = fullmatrix)."""
    out = _dev.empty(((r + 1) * D,))
    dperm = _dev.to_dev(perm, dtype=np.int64) if perm is not None else None
    call("rp_theta_export", ptr(theta_dev), d, r, ptr(dperm), D, ptr(out), stream())
    return out.cpu().numpy().reshape(r + 1, D)


def import_theta(theta, d, r, perm):
    """Reference-layout (r+1, D) coefficients -> device tile layout."""
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    D = theta.shape[1]
    vec = _dev.to_dev(theta)
    out = _dev.empty((tile_elems(d, r + 1),))
    dperm = _dev.to_dev(perm, dtype=np.int64) if perm is not None else None
    call("rp_theta_import", ptr(vec), d, r, ptr(dperm), D, ptr(out), stream())
    return out


def holdout(B, X_val, Y_val, metric):
    """Hold-out error of solution columns B (d, c) against (X_val, Y_val (n, c)) per column."""
    torch = _dev.torch()
    X_val = np.asarray(X_val, dtype=np.float64)
    nv, d = X_val.shape
    B = np.asarray(B, dtype=np.float64).reshape(d, -1)
    c = B.shape[1]
    Y2 = np.asarray(Y_val, dtype=np.float64).reshape(nv, c)
    ldw = c + (c & 1)
    W = _dev.zeros((d, ldw))
    W[:, :c].copy_(torch.from_numpy(np.ascontiguousarray(B)))
    dX = _dev.to_dev(X_val)
    dY = _dev.to_dev(Y2)
    curves = _dev.empty((c,))
    ws = _dev.workspace(_lib.query("rp_holdout_workspace_size", nv, d, 1, c, 1))
    metric_id = _lib.RP_METRIC_RMSE if metric == "rmse" else _lib.RP_METRIC_MISCLASS
    call("rp_holdout_direct", ptr(dX), d, nv, nv, d, ptr(dY), c, c, ptr(W), ldw, d * ldw, 1, 1, metric_id,
         ptr(curves), ptr(ws), stream())
    return curves.cpu().numpy()
