"""Polynomial interpolation of Cholesky factors along the ridge path, on the B200
(drop-in for ridgepath/pichol.py).

``fit`` keeps the reference's contract (pichol.py:68-140): validation order
and exceptions, sorted samples, the monomial observation matrix with the
COND_LIMIT rescale to [-1, 1], least squares by the normal equations, and the
Frobenius residual. The work runs on the device: the s shifted matrices are
factored together by ``rp_potrf_batched`` and the fit ``theta = P T`` (with
P = (V^T V)^{-1} V^T formed on the host from the same V exactly as the
reference forms (V^T V)^{-1} V^T T) runs in ``rp_fit_tiles``, which writes the
device tile layout directly -- the reference's separate bulk_gather pass
(trivec.py:165-191) is fused away; ``theta`` is exported to the caller's
layout at the end (timed as the "vec" phase).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

from . import _dev, _ops, trivec
from .errors import DegenerateSamples, DimensionMismatch, InsufficientSamples, NotPositiveDefinite, NotSymmetric
from .linalg import CholeskyFactor, cholesky

# raw-basis condition number beyond which samples are rescaled to [-1, 1] (pichol.py:25)
COND_LIMIT = 1e8


@dataclass
class InterpModel:
    """Per-entry polynomial coefficients fitted over a lambda window (pichol.py:28-52).

    theta has shape (r+1, D) in ``layout`` order, constant term first, in the
    basis t = t_scale * lambda + t_shift. ``_tiles`` caches the device tile
    layout of theta (filled by ``fit``; rebuilt from theta when absent).
    """

    degree: int
    sample_lambdas: np.ndarray
    theta: np.ndarray
    layout: trivec.VecLayout
    cond_V: float
    t_scale: float
    t_shift: float
    residual_fro: float
    _tiles: object = field(default=None, repr=False, compare=False)

    @property
    def num_samples(self):
        return self.sample_lambdas.shape[0]

    def eval_ops(self):
        """Multiply-add count of one Horner evaluation: degree * D."""
        return self.degree * self.layout.length

    def tiles(self):
        """Device tile-layout coefficients (imported from ``theta`` on first use)."""
        if self._tiles is None:
            lay = self.layout
            self._tiles = _ops.import_theta(self.theta, lay.h, self.degree, lay.perm)
        return self._tiles


@dataclass
class FitDiagnostics:
    """Interpolation error of a model against exact factorization (pichol.py:55-61)."""

    nrmse_per_lambda: dict
    max_nrmse: float
    residual_fro: float


def _observation_matrix(t, r):
    return np.vander(t, r + 1, increasing=True)


def fit_basis(sample_lambdas, r, raw_monomials=False, cond_limit=None):
    """Host half of pichol.fit (pichol.py:103, 112-124).

    Returns (sorted lambdas, V, cond_raw, t_scale, t_shift, P) with
    P = (V^T V)^{-1} V^T computed through the same Cholesky of V^T V and the
    same two triangular solves the reference applies to V^T T.
    """
    if cond_limit is None:
        cond_limit = COND_LIMIT
    lams = np.sort(np.asarray(sample_lambdas, dtype=float))
    V_raw = _observation_matrix(lams, r)
    cond_raw = float(np.linalg.cond(V_raw))
    t_scale, t_shift = 1.0, 0.0
    V = V_raw
    if not raw_monomials and cond_raw > cond_limit:
        span = lams[-1] - lams[0]
        t_scale = 2.0 / span
        t_shift = -(lams[-1] + lams[0]) / span
        V = _observation_matrix(t_scale * lams + t_shift, r)
    VtV = V.T @ V
    try:
        Lv = scipy.linalg.cholesky(VtV, lower=True, check_finite=False)
    except scipy.linalg.LinAlgError as e:
        raise NotPositiveDefinite(str(e)) from e
    w = scipy.linalg.solve_triangular(Lv, V.T, lower=True, check_finite=False)
    P = scipy.linalg.solve_triangular(Lv.T, w, lower=False, check_finite=False)
    return lams, V, cond_raw, t_scale, t_shift, P


def _validate(lams, r):
    g = lams.shape[0]
    if g <= r:
        raise InsufficientSamples(f"need more samples than the degree: g={g}, r={r}")
    if np.unique(lams).shape[0] != g:
        raise DegenerateSamples("sample lambdas must be distinct")
    if np.any(lams <= 0):
        raise DegenerateSamples("sample lambdas must be positive")


def fit(H, sample_lambdas, r, layout, raw_monomials=False, timings=None):
    """Fit the per-entry polynomials from g exact factorizations (pichol.py:68-140)."""
    H = np.asarray(H, dtype=float)
    lams = np.asarray(sample_lambdas, dtype=float)
    _validate(lams, r)
    if H.shape[0] != layout.h:
        raise DimensionMismatch(f"H order {H.shape[0]} vs layout order {layout.h}")
    linalg_check = H.ndim == 2 and H.shape[0] == H.shape[1]
    if not linalg_check:
        raise DimensionMismatch(f"expected a square matrix, got shape {H.shape}")
    torch = _dev.torch()
    lams_sorted, V, cond_raw, t_scale, t_shift, P = fit_basis(lams, r, raw_monomials)
    d = H.shape[0]
    s = lams_sorted.shape[0]

    t0 = time.perf_counter()
    # linalg.cholesky's symmetry check (linalg.py:93-96) on every H + lam*I, in closed form:
    # ||H + lam I||_F^2 = ||H||_F^2 + 2 lam tr(H) + d lam^2 and the asymmetry does not depend on lam.
    asym = np.linalg.norm(H - H.T)
    h2, tr = float(np.sum(H * H)), float(np.trace(H))
    for lam in lams_sorted:
        nrm = np.sqrt(max(h2 + 2.0 * lam * tr + d * lam * lam, 0.0))
        if asym > 1e-10 * max(nrm, 1e-300):
            raise NotSymmetric(f"matrix is not symmetric: ||A - A.T|| = {asym:.3e}")
    dH = _dev.colmajor_to_dev(H).reshape(-1)
    A = dH.repeat(s).reshape(s, d * d)
    diag = torch.arange(d, device=A.device) * (d + 1)
    A[:, diag] += _dev.to_dev(lams_sorted)[:, None]
    info = _ops.potrf(A, d, s)
    if np.any(info != 0):
        i = int(np.flatnonzero(info)[0])
        raise NotPositiveDefinite(
            f"leading minor of order {int(info[i])} is not positive definite at lambda={lams_sorted[i]}"
        )
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    tiles, resid = _ops.fit_tiles(A, d, s, 1, r, P, V)
    residual = float(resid.cpu().numpy()[0])
    t2 = time.perf_counter()
    D = layout.length
    theta = _ops.export_theta(tiles[0], d, r, layout.perm, D)
    t3 = time.perf_counter()
    if timings is not None:
        timings["factorize"] += t1 - t0
        timings["fit"] += t2 - t1
        timings["vec"] += t3 - t2
    return InterpModel(
        degree=r,
        sample_lambdas=lams_sorted,
        theta=theta,
        layout=layout,
        cond_V=cond_raw,
        t_scale=t_scale,
        t_shift=t_shift,
        residual_fro=residual,
        _tiles=tiles[0],
    )


def eval_vector(model, lambda_t):
    """Horner evaluation of all D entry polynomials at one lambda (pichol.py:143-151),
    on the device, in the model's layout order."""
    torch = _dev.torch()
    t = model.t_scale * lambda_t + model.t_shift
    theta = np.asarray(model.theta)
    if theta.dtype != np.float64:
        theta = theta.astype(np.float64)
    th = _dev.to_dev(theta)
    v = th[model.degree].clone()
    for i in range(model.degree - 1, -1, -1):
        v.mul_(t)
        v.add_(th[i])
    out = v.cpu().numpy()
    del torch
    return out


def eval(model, lambda_t):
    """Interpolated factor at lambda_t as a dense F-ordered CholeskyFactor (pichol.py:154-164)."""
    if lambda_t <= 0:
        raise DegenerateSamples(f"lambda must be positive, got {lambda_t}")
    lay = model.layout
    t = model.t_scale * lambda_t + model.t_shift
    L = _ops.materialize(model.tiles(), lay.h, model.degree, t)
    return CholeskyFactor(L, lam=lambda_t, interpolated=True)


def sample_indices(q, g):
    """Indices of g near-evenly spaced grid positions including both ends (pichol.py:167-169)."""
    return np.round(np.linspace(0, q - 1, g)).astype(int)


def nrmse(L_interp, L_exact):
    """Frobenius error normalized by the exact factor's entry range (pichol.py:172-177)."""
    A = L_interp.matrix if isinstance(L_interp, CholeskyFactor) else np.asarray(L_interp)
    B = L_exact.matrix if isinstance(L_exact, CholeskyFactor) else np.asarray(L_exact)
    spread = float(B.max() - B.min())
    return float(np.linalg.norm(A - B) / spread)


def diagnostics(model, H, dense_lambdas):
    """NRMSE of the model against exact factorization at each lambda (pichol.py:180-193)."""
    H = np.asarray(H, dtype=float)
    eye = np.eye(H.shape[0])
    per = {}
    for lam in np.asarray(dense_lambdas, dtype=float):
        exact = cholesky(H + lam * eye, lam=lam)
        interp = eval(model, lam)
        per[float(lam)] = nrmse(interp, exact)
    return FitDiagnostics(
        nrmse_per_lambda=per,
        max_nrmse=max(per.values()),
        residual_fro=model.residual_fro,
    )
