"""Shared constructions (restating the reference's tests/helpers.py:6-45)."""

import numpy as np


def make_spd(rng, m, shift=1.0):
    G = rng.standard_normal((m, m))
    return G @ G.T / m + shift * np.eye(m)


def make_spd_spectrum(d, lo, hi, seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    eig = np.logspace(np.log10(lo), np.log10(hi), d)
    return (Q * eig) @ Q.T


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))
