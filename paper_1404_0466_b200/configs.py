"""Seeded synthetic inputs for the BASELINE.json configs c1..c5.

BASELINE.json fixes the shapes and distributions but not the RNG draw order;
this module fixes it so the GPU path, the oracle and the
golden fixtures all see the same arrays. No public dataset is used: c2/c3 only
imitate MNIST's input shape (784 nonnegative inputs, ~19% nonzero) and feed it
through a random degree-2 Maclaurin feature map.

Folds are contiguous blocks of n // k rows (fold f is the validation block),
i.e. ``FoldPlan(k, np.arange(n) // (n // k), seed)``; ``make_folds`` of the
reference permutes rows and is not what BASELINE specifies.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class CvConfig:
    name: str
    n: int
    d: int
    m: int
    k: int
    s: int  # sampled lambdas (``g`` in the reference API)
    r: int  # polynomial degree (``r`` in the reference API)
    q: int
    lo: float
    hi: float
    generator: str  # "powerlaw" | "maclaurin"
    seed: int = 0

    @property
    def D(self):
        return self.d * (self.d + 1) // 2

    @property
    def n_val(self):
        return self.n // self.k

    def scaled(self, **kw):
        """Same config with some fields replaced (parity tests use smaller n/d)."""
        vals = dict(self.__dict__)
        vals.update(kw)
        return CvConfig(**vals)


CONFIGS = {
    "c1": CvConfig("c1", 2000, 256, 1, 5, 4, 2, 31, 1e-3, 1e1, "powerlaw"),
    "c2": CvConfig("c2", 20000, 1024, 10, 5, 4, 2, 100, 1e-4, 1e2, "maclaurin"),
    "c3": CvConfig("c3", 60000, 2048, 10, 5, 5, 2, 200, 1e-4, 1e2, "maclaurin"),
    "c4": CvConfig("c4", 100000, 4096, 10, 8, 5, 2, 200, 1e-4, 1e2, "powerlaw"),
    "c5": CvConfig("c5", 200000, 8192, 16, 8, 6, 3, 500, 1e-5, 1e3, "powerlaw"),
}


def powerlaw(n, d, m, seed=0):
    """c1/c4/c5: X ~ N(0,1) with column j scaled by (1+j)^-0.5,
    Y = X W* + 0.1 N(0,1), W* ~ N(0,1). Draw order: X, W*, noise."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d))
    X *= (1.0 + np.arange(d)) ** -0.5
    W = rng.standard_normal((d, m))
    Y = X @ W
    Y += 0.1 * rng.standard_normal((n, m))
    return X, Y


def maclaurin(n, d, m=10, seed=0, proj_seed=1):
    """c2/c3: 784-dim sparse nonnegative inputs (nonzero w.p. 0.19, U(0,1)),
    random degree-2 Maclaurin features (Rademacher projections, seed 1),
    one-vs-all +/-1 targets from uniform labels 0..9."""
    rng = np.random.default_rng(seed)
    Xin = (rng.random((n, 784)) < 0.19) * rng.random((n, 784))
    labels = rng.integers(0, 10, n)
    Y = np.where(labels[:, None] == np.arange(m), 1.0, -1.0)
    pr = np.random.default_rng(proj_seed)
    O1 = pr.choice([-1.0, 1.0], (784, d))
    O2 = pr.choice([-1.0, 1.0], (784, d))
    X = (Xin @ O1) * (Xin @ O2) / np.sqrt(d)
    return X, Y


def generate(cfg: CvConfig):
    """(X (n, d) C-order f64, Y (n, m) f64) for a config."""
    if cfg.generator == "powerlaw":
        return powerlaw(cfg.n, cfg.d, cfg.m, cfg.seed)
    if cfg.generator == "maclaurin":
        return maclaurin(cfg.n, cfg.d, cfg.m, cfg.seed)
    raise ValueError(cfg.generator)


def contiguous_assignments(n, k):
    return np.arange(n) // (n // k)


def grid_values(cfg: CvConfig):
    """cvsearch.make_grid (cvsearch.py:55-66)."""
    v = np.logspace(np.log10(cfg.lo), np.log10(cfg.hi), cfg.q)
    v[0], v[-1] = cfg.lo, cfg.hi
    return v
