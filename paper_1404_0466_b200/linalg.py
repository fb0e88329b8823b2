"""Cholesky factorization and triangular solves on the B200 (drop-in for ridgepath/linalg.py).

``cholesky`` mirrors linalg.py:66-101 (square check, 1e-10 relative symmetry
check, lower factor, F-ordered result, NotPositiveDefinite on a failed pivot)
but factors with the batched blocked FP64 kernel ``rp_potrf_batched``.
``solve_chol`` mirrors linalg.py:104-128 and runs the fused tile solve
``rp_eval_solve`` with a degree-0 "polynomial" (the factor itself).

The SVD family of the reference (linalg.py:48-63, 131-207) is outside the
north-star path and is not provided.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _ops
from .errors import DimensionMismatch, NotPositiveDefinite, NotSymmetric


@dataclass
class CholeskyFactor:
    """Lower-triangular factor L with L @ L.T equal to the factored matrix (linalg.py:23-45)."""

    matrix: np.ndarray
    lam: float | None = None
    interpolated: bool = False

    @property
    def dim(self):
        return self.matrix.shape[0]


def _check_square_symmetric(A):
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise DimensionMismatch(f"expected a square matrix, got shape {A.shape}")
    nrm = np.linalg.norm(A)
    asym = np.linalg.norm(A - A.T)
    if asym > 1e-10 * max(nrm, 1e-300):
        raise NotSymmetric(f"matrix is not symmetric: ||A - A.T|| = {asym:.3e}")


def cholesky(A, lam=None):
    """Factor a symmetric positive-definite matrix as A = L @ L.T on the GPU.

    Raises DimensionMismatch, NotSymmetric or NotPositiveDefinite exactly where
    linalg.cholesky (linalg.py:90-100) does.
    """
    A = np.asarray(A, dtype=float)
    _check_square_symmetric(A)
    d = A.shape[0]
    dA = _dev.colmajor_to_dev(A).reshape(-1)
    info = _ops.potrf(dA, d, 1)
    if info[0] != 0:
        raise NotPositiveDefinite(f"leading minor of order {int(info[0])} is not positive definite")
    _ops.lower_of(dA, d)
    return CholeskyFactor(_dev.colmajor_to_host(dA, d), lam=lam)


def solve_chol(factor, g):
    """Solve (L @ L.T) theta = g by blocked forward and back substitution on the GPU.

    g may be (h,) or (h, k); the result has g's shape (linalg.py:104-128).
    """
    L = factor.matrix if isinstance(factor, CholeskyFactor) else np.asarray(factor, dtype=float)
    g = np.asarray(g, dtype=float)
    if g.shape[0] != L.shape[0]:
        raise DimensionMismatch(f"factor order {L.shape[0]} vs rhs length {g.shape[0]}")
    d = L.shape[0]
    dL = _dev.colmajor_to_dev(np.tril(L)).reshape(-1)
    tiles = _ops.pack_lower(dL, d)
    W, _ = _ops.eval_solve(tiles, d, 0, g.reshape(d, -1), [0.0])
    return W[0].reshape(g.shape)
