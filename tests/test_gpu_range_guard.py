"""The int8 tensor-core (Ozaki) products against adversarial inputs, the Gram-form hold-out
against cancellation, and every specialised solve instantiation.

* Range guard (rp_ozaki.cuh OZ_RANGE): a row of the sliced operand whose max |a| exceeds 1024x
  its rms trips a device flag, and the same call then computes the product on FP64 DMMA (gated
  kernel, no host sync). Checked: the flag trips on an intra-column outlier and stays clear on
  the BASELINE generators; Gram blocks stay at FP64 level (normalised by sqrt(G_ii G_jj)) on
  outliers, Cauchy, lognormal and sparse columns; full sweeps on such data match the oracle
  through to the argmins (ridge.py:58-60, cvsearch.py:119-120).
* Cancellation: n_val MSE = y^T y - 2 w^T c + w^T G w is recomputed from the direct residual
  where it would lose more than 20 bits (a near-exact fit).
* Every RP_FAST_LIST entry of csrc/rp_solve_fast.cu, forced with rp_set_option("solve_lam").
"""

import numpy as np
import pytest

from oracle import pichol_oracle as orc
from paper_1404_0466_b200 import _dev, _lib, _ops, configs, pichol
from paper_1404_0466_b200._lib import call, ptr, stream
from paper_1404_0466_b200.engine import PicholEngine
from tests.helpers import make_spd_spectrum, rel

pytestmark = pytest.mark.gpu


def normalized_err(G, G_ref):
    s = np.sqrt(np.outer(np.diag(G_ref), np.diag(G_ref)))
    s[s == 0] = 1.0
    return float(np.max(np.abs(np.tril(G) - np.tril(G_ref)) / s))


def gram_guarded(X):
    """rp_gram_blocks with a caller-held workspace: (G host, range guard flag)."""
    n, d = X.shape
    dX = _dev.to_dev(X)
    G = _dev.empty((d, d))
    ws = _dev.workspace(_lib.query("rp_gram_workspace_size", d, n, 1))
    call("rp_gram_blocks", ptr(dX), d, n, 1, d, None, 1, 0, ptr(G), None, ptr(ws), stream())
    flag = int(ws[:4].view(_dev.torch().int32).cpu()[0])
    return _dev.colmajor_to_host(G.reshape(-1), d), flag


def reference_gram(X):
    """X^T X with the exact-ish compensated products (FP64 BLAS result is the reference's)."""
    return X.T @ X


def adversarial(kind, n, d, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d))
    if kind == "outlier":  # one huge entry inside otherwise unit-scale columns
        X[rng.integers(0, n, 6), rng.integers(0, d, 6)] = 1e8
    elif kind == "cauchy":
        X = rng.standard_cauchy((n, d))
    elif kind == "lognormal":
        X = rng.lognormal(0.0, 3.0, (n, d)) * rng.choice([-1.0, 1.0], (n, d))
    elif kind == "sparse":
        X *= rng.random((n, d)) < 0.01
    elif kind == "spike_scale":  # a column whose values span 1e-6..1e6 (max/rms ~ sqrt(n))
        X[:, 3] *= np.logspace(-6, 6, n)
    return X


def fallbacks():
    return int(_lib.query("rp_ozaki_fallbacks"))


@pytest.mark.parametrize("kind,trips", [("outlier", True), ("spike_scale", True), ("cauchy", None),
                                        ("lognormal", None), ("sparse", False), ("gaussian", False)])
def test_gram_guard_and_accuracy(gpu, kind, trips):
    X = adversarial(kind, 3000, 256, seed=len(kind))
    before = fallbacks()
    G, flag = gram_guarded(X)
    if trips is not None:
        assert flag == int(trips), (kind, flag)
    assert fallbacks() - before == flag  # the gated FP64 kernel ran exactly when the guard tripped
    G_ref = reference_gram(X)
    err = normalized_err(G, G_ref)
    # componentwise, relative to sum_k |x_ki x_kj| (what FP64 itself guarantees)
    absx = np.abs(X)
    cw = float(np.max(np.abs(np.tril(G - G_ref)) / np.maximum(np.tril(absx.T @ absx), 1e-300)))
    print(f"{kind}: guard {flag}, normalised Gram error {err:.2e}, componentwise {cw:.2e}")
    # FP64 level: the reference's own GEMM accumulates K = 3000 products (K u = 3.3e-13); the
    # componentwise bound is loose only for entries that are products of tiny values (sparse rows
    # whose nonzeros span a few decades keep ~54 - log2(max/|x|) bits per entry)
    assert err <= 1e-13
    assert cw <= 1e-10


@pytest.mark.parametrize("name,n,d", [("c1", 4000, 256), ("c2", 5000, 1024), ("c4", 12000, 1152)])
def test_guard_stays_clear_on_baseline_generators(gpu, name, n, d):
    """The BASELINE generators keep every product (Gram, Cholesky trailing updates -- d > 768 --
    and the hold-out) on the tensor cores."""
    cfg = configs.CONFIGS[name].scaled(n=n, d=d, q=20)
    X, Y = configs.generate(cfg)
    _, flag = gram_guarded(X)
    assert flag == 0
    grid = configs.grid_values(cfg)
    lams, V, _, ts, tsh, P = pichol.fit_basis(grid[orc.sample_indices(cfg.q, cfg.s)], cfg.r)
    eng = PicholEngine([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, cfg.q, cfg.s, cfg.r, holdout="gram")
    before = fallbacks()
    eng.sweep(_dev.to_dev(X), _dev.to_dev(Y), lams, P, V, ts * grid + tsh)
    assert fallbacks() == before


@pytest.mark.parametrize("kind", ["outlier", "lognormal", "sparse"])
def test_sweep_on_adversarial_data_matches_oracle(gpu, kind):
    n, d, m, k, q, s, r = 2400, 256, 3, 4, 21, 4, 2
    X = adversarial(kind, n, d, seed=7)
    rng = np.random.default_rng(1)
    Y = X @ rng.standard_normal((d, m)) * 1e-3 + rng.standard_normal((n, m))
    grid = orc.make_grid(1e-1, 1e3, q)
    lams, V, _, ts, tsh, P = pichol.fit_basis(grid[orc.sample_indices(q, s)], r)
    eng = PicholEngine([n // k] * k, d, m, q, s, r, holdout="gram")
    curves, mean, best = eng.sweep(_dev.to_dev(X), _dev.to_dev(Y), lams, P, V, ts * grid + tsh)
    ref = orc.grid_search_pichol(X, Y, configs.contiguous_assignments(n, k), k, grid, g=s, r=r)
    assert rel(curves.cpu().numpy(), ref["curves"]) <= 1e-8
    assert np.array_equal(best.cpu().numpy(), ref["best"])


@pytest.mark.parametrize("holdout", ["gram", "direct"])
def test_near_exact_fit_holdout_matches_oracle(gpu, holdout):
    """y = X w* + 1e-9 noise: the Gram form's y^T y - 2 w^T c + w^T G w cancels to ~1e-8 of its
    terms at small lambda; those columns must come from the direct residual (reference arithmetic)."""
    n, d, m, k, q, s, r = 2000, 256, 2, 5, 25, 4, 2
    X, _ = configs.powerlaw(n, d, m, seed=3)
    rng = np.random.default_rng(4)
    Y = X @ rng.standard_normal((d, m)) + 1e-9 * rng.standard_normal((n, m))
    grid = orc.make_grid(1e-3, 1e1, q)
    lams, V, _, ts, tsh, P = pichol.fit_basis(grid[orc.sample_indices(q, s)], r)
    eng = PicholEngine([n // k] * k, d, m, q, s, r, holdout=holdout)
    curves, mean, best = eng.sweep(_dev.to_dev(X), _dev.to_dev(Y), lams, P, V, ts * grid + tsh)
    ref = orc.grid_search_pichol(X, Y, configs.contiguous_assignments(n, k), k, grid, g=s, r=r)
    c = curves.cpu().numpy()
    err = float(np.max(np.abs(c - ref["curves"]) / ref["curves"]))
    print(f"near-exact fit ({holdout}): curve rel err {err:.2e}, rmse range {c.min():.2e}..{c.max():.2e}")
    assert err <= 1e-8
    assert np.array_equal(best.cpu().numpy(), ref["best"])


FAST_LIST = [(1, 3, 16), (1, 3, 8), (10, 3, 2), (10, 3, 3), (10, 3, 4), (10, 3, 6), (10, 3, 8), (10, 3, 9), (10, 3, 10), (10, 3, 11), (10, 3, 12),
             (10, 3, 16),
             (16, 4, 4), (16, 4, 6), (16, 4, 7), (16, 4, 8)]


@pytest.fixture
def solve_lam():
    yield lambda v: call("rp_set_option", b"solve_lam", v)
    call("rp_set_option", b"solve_lam", 0)


@pytest.mark.parametrize("m,P,lam", FAST_LIST)
def test_every_solve_instantiation(gpu, solve_lam, m, P, lam):
    r = P - 1
    d = 200  # 4 tile rows, the last one padded
    q = 2 * lam + 4 if m % 2 == 0 else 2 * lam + 2  # three chunks, the last overlapping its neighbour
    H = make_spd_spectrum(d, 0.3, 30.0, seed=m * 31 + lam)
    rng = np.random.default_rng(m + lam)
    G = rng.standard_normal((d, m))
    grid = np.logspace(-2, 0, q)
    lams = np.logspace(-2, 0, r + 3)
    mod = orc.fit(H, lams, r)
    lams_s, V, cond, ts, tsh, Pm = pichol.fit_basis(lams, r)
    A = _dev.to_dev(np.stack([np.ascontiguousarray((H + l * np.eye(d)).T) for l in lams_s]).reshape(len(lams), -1))
    assert np.all(_ops.potrf(A, d, len(lams)) == 0)
    tiles, _ = _ops.fit_tiles(A, d, len(lams), 1, r, Pm, V)
    solve_lam(lam)
    W, flags = _ops.eval_solve(tiles[0], d, r, G, ts * grid + tsh)
    assert not np.any(flags)
    worst = max(rel(W[j], orc.solve_interp(mod, G, l)) for j, l in enumerate(grid))
    assert worst <= 1e-10, worst


def _holdout_gram_call(G, C, yy, X, Y, W, n_val, d, m, q, nf, dp, ldw):
    """rp_holdout_gram on device copies (G: nf x d x d column-major blocks, C: nf x m x d, W: nf x dp x ldw)."""
    dG, dC, dyy = _dev.to_dev(G), _dev.to_dev(C), _dev.to_dev(yy)
    dX, dY, dW = _dev.to_dev(X), _dev.to_dev(Y), _dev.to_dev(W)
    curves = _dev.empty((nf, q, m))
    ws = _dev.workspace(_lib.query("rp_holdout_workspace_size", n_val, d, q, m, nf))
    call("rp_holdout_gram", ptr(dG), d * d, ptr(dC), m * d, ptr(dyy), n_val, d, m, ptr(dW), ldw, dp * ldw, q, nf,
         ptr(dX), d, n_val, ptr(dY), m, ptr(curves), ptr(ws), stream())
    return curves.cpu().numpy()


def test_holdout_out_of_range_columns_fall_back_per_tile(gpu):
    """Solution vectors whose entries span more than the tensor-core hold-out's 24-bit budget (c5's
    largest lambdas) are recomputed on FP64 DMMA tile by tile, the rest stay on the int8 tensor
    cores: curves equal the all-DMMA path's, and no full fallback is counted."""
    rng = np.random.default_rng(12)
    nf, n_val, d, m, q = 2, 900, 256, 2, 160
    dp, N = d, q * m
    ldw = N
    X = rng.standard_normal((nf * n_val, d)) * (1 + np.arange(d)) ** -0.5
    Y = rng.standard_normal((nf * n_val, m))
    W = np.zeros((nf, dp, ldw))
    W[:, :d] = rng.standard_normal((nf, d, N)) * 1e-2
    wide = [5, 6, 200, 301]  # columns whose entries span ~40 bits: tiles 0, 1 and 2 of 128 columns
    for f in range(nf):
        for c in wide[f:]:
            W[f, :d, c] *= np.logspace(-12, 0, d)[rng.permutation(d)]
    G = np.stack([np.ascontiguousarray((X[f * n_val:(f + 1) * n_val].T @ X[f * n_val:(f + 1) * n_val]).T)
                  for f in range(nf)])
    C = np.stack([(X[f * n_val:(f + 1) * n_val].T @ Y[f * n_val:(f + 1) * n_val]).T for f in range(nf)])
    yy = np.stack([np.sum(Y[f * n_val:(f + 1) * n_val] ** 2, axis=0) for f in range(nf)])
    before = fallbacks()
    got = _holdout_gram_call(G, C, yy, X, Y, W, n_val, d, m, q, nf, dp, ldw)
    assert fallbacks() == before  # only the marked tiles ran on DMMA, not a full fallback
    call("rp_set_option", b"holdout_ozaki", 0)
    try:
        dmma = _holdout_gram_call(G, C, yy, X, Y, W, n_val, d, m, q, nf, dp, ldw)
    finally:
        call("rp_set_option", b"holdout_ozaki", 1)
    ref = np.stack([[orc.holdout_error(W[f, :d, j * m:(j + 1) * m], X[f * n_val:(f + 1) * n_val],
                                       Y[f * n_val:(f + 1) * n_val]) for j in range(q)] for f in range(nf)])
    assert rel(dmma, ref) <= 1e-12
    assert rel(got, ref) <= 1e-12
    cols = np.array(wide)
    err_wide = max(abs(got[f, c // m, c % m] - ref[f, c // m, c % m]) / ref[f, c // m, c % m]
                   for f in range(nf) for c in cols[f:])
    print(f"per-tile fallback: wide-column rel err {err_wide:.2e}")
    assert err_wide <= 1e-13
