"""Headline parity: the device sweep at the FULL BASELINE sizes against fixtures made by the
real reference (tests/golden/make_golden_baseline.py: ridge.assemble + pichol.fit + per-lambda
pichol.eval / linalg.solve_chol / RMSE, cvsearch.py:154-175's fold mean and first argmin).

What is asserted (north_star):
* the selected lambda index of every output (and of the mean over outputs) is identical;
* the per-fold hold-out curves agree within 1e-10 relative (c4's smallest decision margin is
  6.2e-9, so the north_star 1e-8 tolerance alone would not protect the argmin there);
* the interpolated factor L(lambda) of fold 0 at three grid lambdas agrees within
  1e-10 ||L||_F (pichol.py:154-164), from a Gaussian sketch L R, the diagonal and sampled entries.
The achieved errors are printed (pytest -s) so the margin to each bound is on record.
"""

import numpy as np
import pytest

from paper_1404_0466_b200 import _ops, configs, cvsearch
from tests.conftest import golden

pytestmark = pytest.mark.gpu

CURVE_TOL = 1e-10
FACTOR_TOL = 1e-10


def run_config(name):
    g = golden(f"baseline_{name}")
    cfg = configs.CONFIGS[name]
    X, Y = configs.generate(cfg)
    # the inputs are the seeded arrays the fixtures were made from (BLAS-dependent only in Y's
    # and the Maclaurin features' last bits)
    chk = np.array([X.sum(), (X[::97] ** 2).sum(), Y.sum(), (Y ** 2).sum()])
    assert np.allclose(chk, g["checksums"], rtol=1e-11, atol=1e-9), (chk, g["checksums"])
    grid = configs.grid_values(cfg)
    assert np.array_equal(grid, g["grid"])
    sess = cvsearch.CvSession([cfg.n // cfg.k] * cfg.k, cfg.d, cfg.m, grid, g=cfg.s, r=cfg.r)
    curves, best = sess.run(X, Y)
    return g, cfg, sess, curves, best


def curve_error(curves, ref, mask=None):
    ok = np.isfinite(ref) if mask is None else mask
    return float(np.max(np.abs(curves[ok] - ref[ok]) / np.abs(ref[ok])))


def check_factors(g, cfg, sess):
    """Fold 0's device coefficients, materialised at the fixture's lambdas, against the reference's
    pichol.eval sketches."""
    theta0 = sess.engine.theta[0]
    R = np.random.default_rng(7).standard_normal((cfg.d, 4))  # make_golden_baseline.sketch_inputs
    worst = 0.0
    for a, j in enumerate(g["factor_idx"]):
        t = sess.t_scale * g["grid"][j] + sess.t_shift
        L = _ops.materialize(theta0, cfg.d, cfg.r, t)
        fro = float(g["factor_fro"][a])
        # E ||dL R||_F^2 = 4 ||dL||_F^2 for a d x 4 Gaussian R
        est = float(np.linalg.norm(L @ R - g["factor_sketch"][a])) / 2.0 / fro
        dia = float(np.max(np.abs(np.diag(L) - g["factor_diag"][a]))) / fro
        smp = float(np.max(np.abs(L[g["sample_i"], g["sample_j"]] - g["factor_samples"][a]))) / fro
        print(f"{cfg.name} factor at grid {j}: sketch {est:.2e} diag {dia:.2e} samples {smp:.2e} (x ||L||_F)")
        worst = max(worst, est, dia, smp)
        del L
    assert worst <= FACTOR_TOL, worst


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_full_config_matches_reference(gpu, name):
    g, cfg, sess, curves, best = run_config(name)
    err = curve_error(curves, g["per_fold"])
    mean = curves.sum(axis=0) / cfg.k
    print(f"{name}: curves max rel err {err:.2e}; best {best.tolist()}")
    assert err <= CURVE_TOL
    assert np.array_equal(best, g["best"])
    assert int(np.argmin(mean.mean(axis=1))) == int(g["best_of_mean"])
    check_factors(g, cfg, sess)


@pytest.mark.slow
def test_c4_headline_matches_reference(gpu):
    """All 8 folds x 200 lambdas x 10 outputs of the headline config."""
    g, cfg, sess, curves, best = run_config("c4")
    err = curve_error(curves, g["per_fold"])
    mean = curves.sum(axis=0) / cfg.k
    # how much of each output's decision margin the curve error uses
    srt = np.sort(g["mean"], axis=0)
    margin = (srt[1] - srt[0]) / srt[0]
    print(f"c4: curves max rel err {err:.2e}; smallest margin {margin.min():.2e}; best {best.tolist()}")
    assert err <= CURVE_TOL
    assert np.array_equal(best, g["best"])
    assert int(np.argmin(mean.mean(axis=1))) == int(g["best_of_mean"])
    check_factors(g, cfg, sess)


@pytest.mark.slow
def test_c5_fold0_matches_reference(gpu):
    """c5 (d = 8192, 16 outputs, cubic with the [-1, 1] rescale), fold 0 x 500 lambdas. The
    reference's own cubic interpolant collapses for lambda > 65 (its fitted
    min |L_ii| peaks at 8.07 near lambda = 65, then falls to 7e-5 while the exact factor's stays
    >= 13; curves reach 1e74): there both sides evaluate factors whose conditioning amplifies FP64
    rounding, and they agree to 1e-9..1e-8 where the collapse starts (grid 440-449) and only ~1e-3 in
    the blow-up. Curves are compared (north_star tolerance, 1e-8) on the lambdas where the
    reference's fitted min |L_ii| is at least half its running maximum over smaller lambdas (the
    interpolant still tracks the factor); the excluded grid indices are reported, with the error on
    the excluded lambdas whose curve is still within 100x of its minimum."""
    g, cfg, sess, curves, best = run_config("c5")
    ref = g["per_fold"][0]
    finite = np.isfinite(ref)
    md = g["mindiag"][0]
    keep = (md >= 0.5 * np.maximum.accumulate(md)) & np.all(finite, axis=1)
    sane = np.all(finite & (ref < 100 * np.min(np.where(finite, ref, np.inf), axis=0)), axis=1)
    mask = np.repeat(keep[:, None], cfg.m, axis=1)
    err = curve_error(curves[0], ref, mask)
    per_lam = np.max(np.abs(curves[0] - ref) / np.abs(ref), axis=1)
    edge = sane & ~keep
    print(f"c5 fold 0: curves max rel err {err:.2e} on {keep.sum()} of {cfg.q} lambdas "
          f"(median {np.median(per_lam[keep]):.2e}; excluded grid indices {np.flatnonzero(~keep).tolist()}; "
          f"max err on the excluded lambdas with a sane curve {np.max(per_lam[edge], initial=0.0):.2e})")
    assert keep[:440].all() and keep.sum() >= 440
    assert err <= 1e-8
    # fold 0's own argmins (the selection proper averages 8 folds; the reference's c5 sweep takes ~20
    # CPU-minutes per fold, so only fold 0 is pinned). They sit at lambda <= 0.03, where the curves
    # agree to ~1e-12, below the smallest best-to-second gap (output 11: 2.5e-11).
    cref = np.where(finite, ref, np.inf)
    fold0_best = np.argmin(np.where(np.isfinite(curves[0]), curves[0], np.inf), axis=0)
    ref_best = np.argmin(cref, axis=0)
    srt = np.sort(cref, axis=0)
    gap = (srt[1] - srt[0]) / srt[0]
    near = per_lam[: int(ref_best.max()) + 1].max()
    print(f"c5 fold 0: argmins {fold0_best.tolist()} (reference {ref_best.tolist()}); curve error up to the "
          f"largest argmin {near:.2e}; gaps {[float(f'{v:.2e}') for v in gap]}")
    assert near < gap.min()
    assert np.array_equal(fold0_best, ref_best)
    check_factors(g, cfg, sess)
