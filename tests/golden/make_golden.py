"""Generate the golden fixtures by running the REAL reference package.

Run in the build container only (the reference tree does not exist on the GPU
box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports ``ridgepath`` read-only and writes small ``.npz`` files next to this
script. The fixtures pin both the CPU oracle (``oracle/pichol_oracle.py``) and
the CUDA path; they are committed, the reference is not.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from threadpoolctl import threadpool_limits  # noqa: E402

from ridgepath import cvsearch, linalg, pichol, ridge, trivec  # noqa: E402

from paper_1404_0466_b200 import configs  # noqa: E402


def spd(rng, m, shift=1.0):
    G = rng.standard_normal((m, m))
    return G @ G.T / m + shift * np.eye(m)


def spd_spectrum(d, lo, hi, seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    eig = np.logspace(np.log10(lo), np.log10(hi), d)
    return (Q * eig) @ Q.T


def curves_of(report, grid, k):
    per_fold = np.zeros((k, grid.q))
    for row in report.rows:
        if row["fold"] >= 0:
            j = int(np.searchsorted(grid.values, row["lambda"]))
            per_fold[row["fold"], j] = row["error"]
    mean = np.array([report.per_lambda_error[float(l)] for l in grid.values])
    return per_fold, mean


def cv_case(name, X, Y, k, lo, hi, q, g, r, metric=cvsearch.RMSE, exact=False):
    n = X.shape[0]
    assign = np.arange(n) // (n // k)
    folds = cvsearch.FoldPlan(k, assign, 0)
    grid = cvsearch.make_grid(lo, hi, q)
    Y2 = Y.reshape(n, -1)
    m = Y2.shape[1]
    per_fold = np.zeros((k, q, m))
    mean = np.zeros((q, m))
    best = np.zeros(m, dtype=np.int64)
    best_lambda = np.zeros(m)
    best_error = np.zeros(m)
    for j in range(m):
        rep = cvsearch.grid_search_pichol(cvsearch.Dataset(X, Y2[:, j]), grid, folds, metric=metric, g=g, r=r)
        pf, mn = curves_of(rep, grid, k)
        per_fold[:, :, j] = pf
        mean[:, j] = mn
        best[j] = int(np.argmin(mn))
        best_lambda[j] = rep.best_lambda
        best_error[j] = rep.best_error
    out = dict(X=X, Y=Y2, k=k, lo=lo, hi=hi, q=q, g=g, r=r, metric=metric, grid=grid.values,
               per_fold=per_fold, mean=mean, best=best, best_lambda=best_lambda, best_error=best_error)
    if exact:
        ex = np.zeros((q, m))
        for j in range(m):
            rep = cvsearch.grid_search_exact(cvsearch.Dataset(X, Y2[:, j]), grid, folds, metric=metric)
            ex[:, j] = curves_of(rep, grid, k)[1]
        out["exact_mean"] = ex
    return out


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def main():
    with threadpool_limits(limits=1):
        # 1. c1 as specified, full sweep, stock driver (single target)
        c1 = configs.CONFIGS["c1"]
        X, Y = configs.generate(c1)
        case = cv_case("c1", X, Y[:, 0], c1.k, c1.lo, c1.hi, c1.q, c1.s, c1.r, exact=True)
        case.pop("X")
        case.pop("Y")  # regenerated from configs.generate (checked by checksum)
        save("c1_cv", x_sum=X.sum(), y_sum=Y.sum(), **case)

        # 2. small multi-output cv (stock driver once per output column)
        Xs, Ys = configs.powerlaw(360, 24, 3, seed=7)
        save("small_multi_cv", **cv_case("small", Xs, Ys, 3, 1e-3, 1e1, 17, 4, 2, exact=True))

        # 3. small misclassification cv on +/-1 targets (maclaurin features)
        Xm, Ym = configs.maclaurin(400, 32, m=2, seed=3)
        save("small_misclass_cv", **cv_case("mis", Xm, Ym, 4, 1e-3, 1e2, 13, 4, 2, metric=cvsearch.MISCLASS))

        # 4. pichol.fit / eval / solve_interp on a d=40 SPD matrix, recursive h0=8
        rng = np.random.default_rng(2024)
        H = spd(rng, 40)
        gvec = rng.standard_normal(40)
        Gmat = rng.standard_normal((40, 3))
        lams = np.array([0.05, 0.2, 0.7, 2.0])
        eval_lams = np.array([0.05, 0.11, 0.9, 3.5])
        fits = {}
        for kind, h0 in ((trivec.RECURSIVE, 8), (trivec.ROWWISE, 64), (trivec.FULLMATRIX, 64)):
            layout = trivec.build_layout(kind, 40, h0)
            model = pichol.fit(H, lams, 2, layout)
            fits[kind] = dict(
                theta=model.theta, residual_fro=model.residual_fro, cond_V=model.cond_V,
                t_scale=model.t_scale, t_shift=model.t_shift,
                L=np.stack([pichol.eval(model, l).matrix for l in eval_lams]),
                v=np.stack([pichol.eval_vector(model, l) for l in eval_lams]),
            )
        p = ridge.RidgeProblem(X=None, y=None, H=H, g=gvec)
        layout = trivec.build_layout(trivec.RECURSIVE, 40, 8)
        model = pichol.fit(H, lams, 2, layout)
        sol = np.stack([ridge.solve_interp(p, model, l).theta for l in eval_lams])
        res = np.array([ridge.solve_interp(p, model, l).residual for l in eval_lams])
        solm = np.stack([linalg.solve_chol(pichol.eval(model, l), Gmat) for l in eval_lams])
        exact_L = np.stack([linalg.cholesky(H + l * np.eye(40)).matrix for l in lams])
        save("fit_d40", H=H, g=gvec, Gmat=Gmat, lams=lams, eval_lams=eval_lams,
             **{f"{k}_{f}": v for k, d in fits.items() for f, v in d.items()},
             solve_theta=sol, solve_residual=res, solve_multi=solm, exact_L=exact_L)

        # 5. rescale branch (cond(V_raw) > COND_LIMIT), degree 3 fit on a tight window
        H5 = spd(np.random.default_rng(5), 6)
        tight = 1e4 + np.linspace(0.0, 1e-3, 5)
        layout = trivec.build_layout(trivec.ROWWISE, 6)
        m5 = pichol.fit(H5, tight, 2, layout)
        save("fit_rescale", H=H5, lams=tight, theta=m5.theta, cond_V=m5.cond_V, t_scale=m5.t_scale,
             t_shift=m5.t_shift, residual_fro=m5.residual_fro,
             L_mid=pichol.eval(m5, tight[2]).matrix)

        # 6. wide-window cubic fit (c5-like rescale in a log-spread window)
        H6 = spd_spectrum(24, 0.5, 50.0, seed=11)
        grid6 = cvsearch.make_grid(1e-5, 1e3, 41)
        s6 = grid6.values[pichol.sample_indices(41, 6)]
        layout = trivec.build_layout(trivec.RECURSIVE, 24, 4)
        m6 = pichol.fit(H6, s6, 3, layout)
        save("fit_wide_cubic", H=H6, lams=s6, theta=m6.theta, cond_V=m6.cond_V, t_scale=m6.t_scale,
             t_shift=m6.t_shift, residual_fro=m6.residual_fro,
             L=np.stack([pichol.eval(m6, l).matrix for l in grid6.values[::10]]), eval_lams=grid6.values[::10])

        # 7. layout permutations (recursive + rowwise) at several (h, h0)
        perms = {}
        for h, h0 in ((4, 2), (5, 4), (9, 4), (17, 4), (33, 8), (64, 8), (100, 64), (130, 64), (256, 64)):
            perms[f"recursive_{h}_{h0}"] = trivec.build_layout(trivec.RECURSIVE, h, h0).perm
        for h in (1, 3, 7, 64):
            perms[f"rowwise_{h}"] = trivec.build_layout(trivec.ROWWISE, h).perm
        save("layouts", **perms)

        # 8. assemble on a seeded design (Hessian parity)
        Xa, Ya = configs.powerlaw(300, 20, 2, seed=9)
        pa = ridge.assemble(Xa, Ya[:, 0])
        save("assemble", X=Xa, Y=Ya, H=pa.H, g=pa.g)


if __name__ == "__main__":
    main()
