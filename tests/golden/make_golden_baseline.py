"""Golden fixtures for the BASELINE.json configs c2..c5, made by the REAL reference.

Run in the build container only (the reference tree does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_baseline.py c4

The inputs are the seeded arrays of ``paper_1404_0466_b200.configs`` (the GPU test
regenerates them from the same seed; only checksums are stored). Each fold is computed
with the reference's own functions, composed for m outputs as SURVEY.md 8(c)(ii) says:

* ``ridge.assemble(X_tr, y_tr)`` -> H (direct X_tr^T X_tr, symmetrised; ridge.py:50-60),
  and G_f = X_tr^T Y_tr for all m outputs (the same product ridge.py:60 forms per output);
* ``pichol.fit(H, sample_lambdas, r, build_layout("recursive", d, 64))`` (pichol.py:68-140,
  the layout ``grid_search_pichol`` uses, cvsearch.py:206-243);
* per grid lambda: ``pichol.eval`` (pichol.py:154-164), the singular check of
  ``ridge.solve_interp`` (ridge.py:88-89), ``linalg.solve_chol(L, G_f)`` (linalg.py:104-128)
  and the RMSE of ``cvsearch.holdout_error`` (cvsearch.py:119-120) per output column;
* fold mean ``np.mean`` over folds (cvsearch.py:156) and first argmin (cvsearch.py:164).

For fold 0 at three grid lambdas it also stores sketches of the interpolated factor
(L @ R for a seeded Gaussian R, the diagonal, ||L||_F and sampled lower entries), so the
device factor can be checked against 1e-10 ||L||_F without committing d x d matrices.
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from threadpoolctl import threadpool_limits  # noqa: E402

from ridgepath import cvsearch, linalg, pichol, ridge, trivec  # noqa: E402

from paper_1404_0466_b200 import configs  # noqa: E402

# grid indices whose interpolated factors are sketched (fold 0); none is a sample point
FACTOR_IDX = {"c2": (17, 50, 80), "c3": (25, 66, 175), "c4": (25, 66, 175), "c5": (50, 211, 350)}
FOLDS = {"c5": (0,)}  # c5: fold 0 only (~20 min of CPU per fold)
SKETCH_COLS = 4
N_SAMPLES = 4096


def sketch_inputs(d, seed=7):
    rng = np.random.default_rng(seed)
    R = rng.standard_normal((d, SKETCH_COLS))
    i = rng.integers(0, d, N_SAMPLES)
    j = rng.integers(0, d, N_SAMPLES)
    return R, np.maximum(i, j), np.minimum(i, j)


def checksums(X, Y):
    """Generator drift detectors: exact-ish sums the GPU test recomputes."""
    return np.array([X.sum(), (X[::97] ** 2).sum(), Y.sum(), (Y ** 2).sum()])


def run(name):
    cfg = configs.CONFIGS[name]
    t0 = time.perf_counter()
    X, Y = configs.generate(cfg)
    n, d, m, k, q = cfg.n, cfg.d, cfg.m, cfg.k, cfg.q
    print(f"{name}: generated in {time.perf_counter() - t0:.1f}s", flush=True)
    assign = configs.contiguous_assignments(n, k)
    grid = cvsearch.make_grid(cfg.lo, cfg.hi, q)
    sample_lams = grid.values[pichol.sample_indices(q, cfg.s)]
    folds = FOLDS.get(name, tuple(range(k)))
    R, si, sj = sketch_inputs(d)
    fidx = FACTOR_IDX[name]

    per_fold = np.full((k, q, m), np.nan)
    mindiag = np.full((k, q), np.nan)
    fac_sketch = np.zeros((len(fidx), d, SKETCH_COLS))
    fac_diag = np.zeros((len(fidx), d))
    fac_fro = np.zeros(len(fidx))
    fac_samples = np.zeros((len(fidx), N_SAMPLES))
    model_info = []
    for f in folds:
        t1 = time.perf_counter()
        val = assign == f
        X_tr, Y_tr, X_val, Y_val = X[~val], Y[~val], X[val], Y[val]
        sub = ridge.assemble(X_tr, Y_tr[:, 0])
        G = X_tr.T @ Y_tr
        del X_tr
        layout = trivec.build_layout(trivec.RECURSIVE, d, 64)
        model = pichol.fit(sub.H, sample_lams, cfg.r, layout)
        model_info.append([model.cond_V, model.t_scale, model.t_shift, model.residual_fro])
        t2 = time.perf_counter()
        for j, lam in enumerate(grid.values):
            L = pichol.eval(model, lam)
            md = float(np.min(np.abs(np.diag(L.matrix))))
            mindiag[f, j] = md
            if f == folds[0] and j in fidx:
                a = fidx.index(j)
                Lm = L.matrix
                fac_sketch[a] = Lm @ R
                fac_diag[a] = np.diag(Lm)
                fac_fro[a] = np.linalg.norm(Lm)
                fac_samples[a] = Lm[si, sj]
            if md < 1e-12:  # ridge.solve_interp raises SingularInterpolant here
                continue
            W = linalg.solve_chol(L, G)
            pred = X_val @ W
            per_fold[f, j] = np.sqrt(np.mean((pred - Y_val) ** 2, axis=0))
        print(f"{name} fold {f}: setup {t2 - t1:.1f}s sweep {time.perf_counter() - t2:.1f}s", flush=True)

    out = dict(n=n, d=d, m=m, k=k, q=q, s=cfg.s, r=cfg.r, lo=cfg.lo, hi=cfg.hi, grid=grid.values,
               folds=np.array(folds), per_fold=per_fold, mindiag=mindiag,
               model_info=np.array(model_info), checksums=checksums(X, Y),
               factor_idx=np.array(fidx), factor_sketch=fac_sketch, factor_diag=fac_diag,
               factor_fro=fac_fro, factor_samples=fac_samples, sample_i=si, sample_j=sj)
    if len(folds) == k:
        mean = np.mean(per_fold, axis=0)  # cvsearch.py:156 (row-sequential over folds)
        out["mean"] = mean
        out["best"] = np.argmin(mean, axis=0)  # cvsearch.py:164, per output
        out["best_of_mean"] = int(np.argmin(mean.mean(axis=1)))
        srt = np.sort(mean, axis=0)
        out["gap"] = (srt[1] - srt[0]) / srt[0]
    path = os.path.join(HERE, f"baseline_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: wrote {path} in {time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    with threadpool_limits(int(os.environ.get("GOLDEN_THREADS", os.cpu_count()))):
        for name in sys.argv[1:] or ["c2", "c3", "c4", "c5"]:
            run(name)
