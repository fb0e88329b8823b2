"""Ridge normal equations on the B200 (drop-in for the hot-path half of ridgepath/ridge.py).

``assemble`` (ridge.py:50-60) builds H = X^T X and g = X^T y with the DMMA Gram
kernel (only the lower tiles are computed; the mirror makes H exactly
symmetric, which is what the reference's 0.5 (H + H^T) guarantees).
``solve_interp`` (ridge.py:78-91) evaluates the fitted factor polynomials and
solves in one fused kernel (``rp_eval_solve``), raising SingularInterpolant at
the same 1e-12 diagonal threshold. ``solve_exact`` (ridge.py:69-75) is the
exact-Cholesky comparator.

Multi-output generalization: y may be (n, m); g is then (d, m) and solutions
are (d, m). The reference is single-target (ridge.py:53 flattens y).
The SVD backends (ridge.py:94-124) are outside the north-star path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _ops, linalg, pichol
from .errors import DegenerateSamples, DimensionMismatch, NotPositiveDefinite, SingularInterpolant

CHOL = "chol"
PICHOL = "pichol"
SVD = "svd"
TSVD = "tsvd"
RSVD = "rsvd"


@dataclass
class RidgeProblem:
    """A design matrix with cached normal-equation pieces (ridge.py:24-39)."""

    X: np.ndarray
    y: np.ndarray
    H: np.ndarray
    g: np.ndarray

    @property
    def n(self):
        return self.X.shape[0]

    @property
    def dim(self):
        return self.H.shape[0]


@dataclass
class Solution:
    theta: np.ndarray
    lam: float
    backend: str
    residual: float


def assemble(X, y):
    """Build a RidgeProblem, caching H = X.T X and g = X.T y (ridge.py:50-60)."""
    X = np.asarray(X, dtype=float)
    y = np.asarray(y, dtype=float)
    if y.ndim != 2:
        y = y.reshape(-1)
    if X.ndim != 2:
        raise DimensionMismatch(f"design matrix must be 2-D, got ndim={X.ndim}")
    if X.shape[0] != y.shape[0]:
        raise DimensionMismatch(f"{X.shape[0]} rows vs {y.shape[0]} targets")
    G, C = _ops.gram(X, y)
    d = X.shape[1]
    H = _dev.colmajor_to_host(G.reshape(-1), d)
    g = C.cpu().numpy().T  # (d, m)
    g = g[:, 0].copy() if y.ndim == 1 else np.ascontiguousarray(g)
    return RidgeProblem(X=X, y=y, H=H, g=g)


def _device_H(p):
    """p.H on the device, uploaded once per RidgeProblem (d x d: 134 MB at d = 4096, ~2.5 ms of PCIe per
    upload) and reused by every solve_* call on it. The copy is re-uploaded when p.H is replaced or
    when a sample of its entries changed in place."""
    H = np.asarray(p.H, dtype=float)
    flat = H.reshape(-1)
    probe = flat[:: max(1, flat.size // 61)].copy()
    key = (id(p.H), H.__array_interface__["data"][0], H.shape)
    cached = getattr(p, "_H_dev", None)
    if cached is None or cached[0] != key or not np.array_equal(cached[1], probe):
        cached = (key, probe, _dev.to_dev(H))
        object.__setattr__(p, "_H_dev", cached)
    return cached[2]


def _certify(p, lam, theta, backend):
    """Relative normal-equation residual ||H theta + lam theta - g|| / ||g|| (ridge.py:63-66)."""
    torch = _dev.torch()
    H = _device_H(p)
    th = _dev.to_dev(theta)
    g = _dev.to_dev(p.g)
    res = float(torch.linalg.norm(H @ th + lam * th - g))
    gn = float(np.linalg.norm(p.g))
    return Solution(theta=theta, lam=float(lam), backend=backend, residual=float(res / max(gn, 1e-300)))


def solve_exact(p, lam):
    """Factor H + lambda*I and solve by substitution (ridge.py:69-75)."""
    if lam < 0:
        raise NotPositiveDefinite(f"negative ridge {lam}")
    L = linalg.cholesky(p.H + lam * np.eye(p.dim), lam=lam)
    theta = linalg.solve_chol(L, p.g)
    return _certify(p, lam, theta, CHOL)


def solve_interp(p, model, lam):
    """Solve with an interpolated factor in place of an exact one (ridge.py:78-91).

    Raises SingularInterpolant when a fitted diagonal has collapsed below 1e-12
    at this lambda; never touches p.X.
    """
    if lam <= 0:
        raise DegenerateSamples(f"lambda must be positive, got {lam}")
    g = np.asarray(p.g, dtype=float)
    d = model.layout.h
    if g.shape[0] != d:
        raise DimensionMismatch(f"factor order {d} vs rhs length {g.shape[0]}")
    t = model.t_scale * lam + model.t_shift
    W, flags = _ops.eval_solve(model.tiles(), d, model.degree, g.reshape(d, -1), [t])
    if flags[0]:
        raise SingularInterpolant(f"interpolated factor is singular at lambda={lam}")
    theta = W[0].reshape(g.shape)
    return _certify(p, lam, theta, PICHOL)


__all__ = ["RidgeProblem", "Solution", "assemble", "solve_exact", "solve_interp", "pichol", "CHOL", "PICHOL"]
