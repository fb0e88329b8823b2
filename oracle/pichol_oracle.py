"""CPU oracle for the piCholesky cross-validation path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it. The product package
(``paper_1404_0466_b200``) never imports anything under ``oracle/`` and
fails loudly when its CUDA library is missing.

It is a numpy/scipy restatement of the reference package ``ridgepath``
(``/root/reference/pkg/src/ridgepath``), following the reference line by
line for the hot path ``cvsearch.grid_search_pichol`` (cvsearch.py:206-243):

* ``make_grid``          -> cvsearch.py:55-66
* ``sample_indices``     -> pichol.py:167-169
* ``contiguous_folds``   -> FoldPlan cvsearch.py:69-73, _fold_slices :145-147
* ``assemble``           -> ridge.py:50-60 (multi-output: Y is (n, m))
* ``cholesky``           -> linalg.py:66-101 (LAPACK dpotrf via scipy)
* ``solve_chol``         -> linalg.py:104-128 (two dtrtrs)
* ``rowwise_perm`` / ``recursive_perm`` -> trivec.py:41-62
* ``fit``                -> pichol.py:68-140 (normal equations, COND_LIMIT rescale)
* ``eval_vector``        -> pichol.py:143-151 (Horner)
* ``eval_dense``         -> pichol.py:154-164 + trivec.unvectorize trivec.py:150-162
* ``solve_interp``       -> ridge.py:78-91 (SingularInterpolant threshold 1e-12)
* ``holdout_error``      -> cvsearch.py:106-123 (RMSE / MISCLASS)
* ``merge``              -> cvsearch.py:154-175 (np.mean over folds, first argmin)
* ``grid_search_pichol`` -> cvsearch.py:206-243, the multi-RHS composition of
  SURVEY.md 8(c): one fit per fold, then per lambda eval + solve_chol with the
  d x m right-hand side and per-column hold-out error. For m == 1 it is the
  stock reference driver's arithmetic.

Parity is pinned: ``tests/golden/make_golden.py`` imports the real reference
(read-only, in the build container only) and writes the fixtures under
``tests/golden/``; ``tests/test_oracle_golden.py`` checks this module against
them.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

COND_LIMIT = 1e8  # pichol.py:25
SINGULAR_DIAG = 1e-12  # ridge.py:88
RMSE = "rmse"  # cvsearch.py:29
MISCLASS = "misclass"  # cvsearch.py:30


class OracleError(Exception):
    """Raised where the reference raises one of its errors.py exceptions."""

    def __init__(self, kind, msg=""):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ---------------------------------------------------------------- grid / folds


def make_grid(lo, hi, q):
    """cvsearch.py:55-66: q log-spaced values, endpoints pinned."""
    if not (0 < lo < hi):
        raise OracleError("UsageError", f"need 0 < lo < hi, got {lo}, {hi}")
    if q < 1:
        raise OracleError("UsageError", f"grid size must be >= 1, got {q}")
    if q == 1:
        return np.array([lo])
    v = np.logspace(np.log10(lo), np.log10(hi), q)
    v[0], v[-1] = lo, hi
    return v


def sample_indices(q, g):
    """pichol.py:167-169 (np.round is half-to-even)."""
    return np.round(np.linspace(0, q - 1, g)).astype(int)


def contiguous_assignments(n, k):
    """BASELINE folds: contiguous blocks of n // k rows."""
    return np.arange(n) // (n // k)


# ---------------------------------------------------------------- primitives


def assemble(X, Y):
    """ridge.py:50-60: H = X^T X symmetrized (:58-59), G = X^T Y (:60)."""
    X = np.asarray(X, dtype=float)
    Y = np.asarray(Y, dtype=float)
    H = X.T @ X
    H = 0.5 * (H + H.T)
    return H, X.T @ Y


def cholesky(A):
    """linalg.py:90-101: symmetry check at 1e-10 relative, dpotrf lower."""
    A = np.asarray(A, dtype=float)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise OracleError("DimensionMismatch", f"shape {A.shape}")
    nrm = np.linalg.norm(A)
    asym = np.linalg.norm(A - A.T)
    if asym > 1e-10 * max(nrm, 1e-300):
        raise OracleError("NotSymmetric", f"{asym:.3e}")
    try:
        L = scipy.linalg.cholesky(A, lower=True, check_finite=False)
    except scipy.linalg.LinAlgError as e:
        raise OracleError("NotPositiveDefinite", str(e)) from e
    return np.asfortranarray(L)


def solve_chol(L, G):
    """linalg.py:104-128: forward then back substitution (dtrtrs x2)."""
    w = scipy.linalg.solve_triangular(L, G, lower=True, check_finite=False)
    return scipy.linalg.solve_triangular(L.T, w, lower=False, check_finite=False)


def rowwise_perm(h):
    """trivec.py:41-43: row-major lower triangle into column-major h x h."""
    p, q = np.tril_indices(h)
    return q * h + p


def recursive_perm(h, h0):
    """trivec.py:46-62: off-diagonal square block first (column-major), then
    the two diagonal triangles, base case rowwise at order <= h0."""
    out = []

    def rec(r0, c0, n):
        if n <= h0:
            p, q = np.tril_indices(n)
            out.append((c0 + q) * h + (r0 + p))
            return
        m = (n + 1) // 2
        rows = np.arange(r0 + m, r0 + n)
        cols = np.arange(c0, c0 + m)
        out.append((cols[:, None] * h + rows[None, :]).reshape(-1))
        rec(r0, c0, m)
        rec(r0 + m, c0 + m, n - m)

    rec(0, 0, h)
    return np.concatenate(out)


# ---------------------------------------------------------------- pichol fit / eval


def vandermonde(t, r):
    """pichol.py:64-65."""
    return np.vander(t, r + 1, increasing=True)


def fit_basis(sample_lambdas, r, raw_monomials=False, cond_limit=COND_LIMIT):
    """pichol.py:103,112-120: sorted samples, cond of the raw basis, and the
    [-1, 1] rescale decision. Returns (lams, V, cond_raw, t_scale, t_shift)."""
    lams = np.sort(np.asarray(sample_lambdas, dtype=float))
    V_raw = vandermonde(lams, r)
    cond_raw = float(np.linalg.cond(V_raw))
    t_scale, t_shift = 1.0, 0.0
    V = V_raw
    if not raw_monomials and cond_raw > cond_limit:
        span = lams[-1] - lams[0]
        t_scale = 2.0 / span
        t_shift = -(lams[-1] + lams[0]) / span
        V = vandermonde(t_scale * lams + t_shift, r)
    return lams, V, cond_raw, t_scale, t_shift


def fit(H, sample_lambdas, r, perm=None, raw_monomials=False):
    """pichol.py:68-140. Returns a dict with theta (r+1, D) packed by ``perm``
    (default: rowwise), T, cond_V, t_scale, t_shift, residual_fro."""
    H = np.asarray(H, dtype=float)
    lams0 = np.asarray(sample_lambdas, dtype=float)
    g = lams0.shape[0]
    if g <= r:
        raise OracleError("InsufficientSamples", f"g={g}, r={r}")
    if np.unique(lams0).shape[0] != g:
        raise OracleError("DegenerateSamples", "not distinct")
    if np.any(lams0 <= 0):
        raise OracleError("DegenerateSamples", "not positive")
    h = H.shape[0]
    if perm is None:
        perm = rowwise_perm(h)
    lams, V, cond_raw, t_scale, t_shift = fit_basis(lams0, r, raw_monomials)
    eye = np.eye(h)
    factors = [cholesky(H + lam * eye) for lam in lams]  # pichol.py:105-107
    T = np.stack([f.reshape(-1, order="F")[perm] for f in factors])  # trivec.bulk_gather
    G = V.T @ T  # pichol.py:122
    Lv = cholesky(V.T @ V)  # pichol.py:123
    theta = solve_chol(Lv, G)  # pichol.py:124
    residual = float(np.linalg.norm(T - V @ theta))  # pichol.py:125
    return dict(
        degree=r,
        sample_lambdas=lams,
        theta=theta,
        T=T,
        perm=perm,
        h=h,
        cond_V=cond_raw,
        t_scale=t_scale,
        t_shift=t_shift,
        residual_fro=residual,
        factors=factors,
    )


def eval_vector(model, lam):
    """pichol.py:143-151: Horner, exactly r*D mul+add."""
    t = model["t_scale"] * lam + model["t_shift"]
    theta = model["theta"]
    v = theta[model["degree"]].copy()
    for i in range(model["degree"] - 1, -1, -1):
        v *= t
        v += theta[i]
    return v


def eval_dense(model, lam):
    """pichol.py:154-164 + trivec.py:150-162: scatter into zeroed F-order h x h."""
    if lam <= 0:
        raise OracleError("DegenerateSamples", f"lambda {lam}")
    h = model["h"]
    flat = np.zeros(h * h)
    flat[model["perm"]] = eval_vector(model, lam)
    return flat.reshape((h, h), order="F")


def solve_interp(model, G, lam):
    """ridge.py:78-91 minus the discarded certificate: eval, singular check,
    solve_chol with the (h,) or (h, m) right-hand side."""
    L = eval_dense(model, lam)
    if np.min(np.abs(np.diag(L))) < SINGULAR_DIAG:
        raise OracleError("SingularInterpolant", f"lambda={lam}")
    return solve_chol(L, G)


# ---------------------------------------------------------------- hold-out / merge


def holdout_error(B, X_val, Y_val, metric=RMSE):
    """cvsearch.py:106-123, per output column: RMSE sqrt(mean((X B - Y)^2))
    or MISCLASS mean(sign mismatch with pred >= 0 -> +1)."""
    X_val = np.asarray(X_val, dtype=float)
    if X_val.shape[0] == 0:
        raise OracleError("EmptyValidationSet", "")
    pred = X_val @ B
    Y_val = np.asarray(Y_val, dtype=float).reshape(pred.shape)
    if metric == RMSE:
        return np.sqrt(np.mean((pred - Y_val) ** 2, axis=0))
    if metric == MISCLASS:
        return np.mean(np.where(pred >= 0, 1.0, -1.0) != np.sign(Y_val), axis=0)
    raise OracleError("UsageError", f"metric {metric!r}")


def merge(fold_curves):
    """cvsearch.py:156,164: np.mean over folds (row-sequential), first argmin.
    fold_curves: (k, q) or (k, q, m). Returns (mean curve, best index per output)."""
    errs = np.mean(np.asarray(fold_curves), axis=0)
    best = np.argmin(errs, axis=0)
    return errs, best


# ---------------------------------------------------------------- the hot path


def grid_search_pichol(X, Y, assignments, k, grid, g=4, r=2, metric=RMSE,
                       raw_monomials=False, folds=None, lam_idx=None):
    """cvsearch.py:206-243, multi-RHS composition.

    Y may be (n,) or (n, m). ``folds`` limits the folds computed and
    ``lam_idx`` the grid points evaluated (bounded CPU samples for bench.py).
    Returns dict(curves (k', q', m), mean (q', m) when all folds/lambdas are
    computed, best (m,), models).
    """
    X = np.asarray(X, dtype=float)
    Y = np.asarray(Y, dtype=float)
    if Y.ndim == 1:
        Y = Y[:, None]
    grid = np.asarray(grid, dtype=float)
    q = grid.shape[0]
    if g > q:
        raise OracleError("UsageError", f"g={g} > q={q}")
    sample_lams = grid[sample_indices(q, g)]  # cvsearch.py:223
    folds = list(range(k)) if folds is None else list(folds)
    lam_idx = np.arange(q) if lam_idx is None else np.asarray(lam_idx)
    curves = []
    models = []
    for i in folds:
        val = assignments == i  # cvsearch.py:145-147
        H, G = assemble(X[~val], Y[~val])
        model = fit(H, sample_lams, r, raw_monomials=raw_monomials)
        models.append(model)
        errs = np.empty((lam_idx.shape[0], Y.shape[1]))
        for j, li in enumerate(lam_idx):
            B = solve_interp(model, G, grid[li])
            errs[j] = holdout_error(B, X[val], Y[val], metric)
        curves.append(errs)
    curves = np.stack(curves)
    out = dict(curves=curves, models=models, sample_lambdas=sample_lams)
    if len(folds) == k and lam_idx.shape[0] == q:
        mean, best = merge(curves)
        out["mean"] = mean
        out["best"] = best
    return out


def grid_search_exact(X, Y, assignments, k, grid, metric=RMSE):
    """cvsearch.py:178-203: one exact factorization per fold per grid point
    (linalg.cholesky of H + lam I, solve_chol, holdout_error). Returns dict(curves (k, q, m),
    mean (q, m), best (m,))."""
    X = np.asarray(X, dtype=float)
    Y = np.asarray(Y, dtype=float)
    if Y.ndim == 1:
        Y = Y[:, None]
    grid = np.asarray(grid, dtype=float)
    curves = np.empty((k, grid.shape[0], Y.shape[1]))
    for i in range(k):
        val = assignments == i
        H, G = assemble(X[~val], Y[~val])
        eye = np.eye(H.shape[0])
        for j, lam in enumerate(grid):
            B = solve_chol(cholesky(H + lam * eye), G)
            curves[i, j] = holdout_error(B, X[val], Y[val], metric)
    mean, best = merge(curves)
    return dict(curves=curves, mean=mean, best=best)
