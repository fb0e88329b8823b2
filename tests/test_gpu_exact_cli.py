"""Device exact-Cholesky CV (cvsearch.grid_search_exact, cvsearch.py:178-203; mchol_search
:246-320; pinrmse_search :322-380) and the command line (cli.py) against the reference's golden
fixtures and the CPU oracle.

Tolerances as for the piCholesky sweep: hold-out errors within 1e-8 relative, misclass
error rates identical, identical selected lambda."""

import csv
import json
import os

import numpy as np
import pytest

from oracle import pichol_oracle as orc
from paper_1404_0466_b200 import cli, configs, cvsearch, exact
from paper_1404_0466_b200.errors import NotPositiveDefinite, UsageError
from tests.conftest import golden
from tests.helpers import rel

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "cli")


def curve_of(report, grid):
    return np.array([report.per_lambda_error[float(l)] for l in grid.values])


@pytest.mark.parametrize("holdout", ["gram", "direct"])
def test_exact_c1_matches_reference(gpu, holdout):
    g = golden("c1_cv")
    c1 = configs.CONFIGS["c1"]
    X, Y = configs.generate(c1)
    grid = cvsearch.make_grid(c1.lo, c1.hi, c1.q)
    rep = cvsearch.grid_search_exact(cvsearch.Dataset(X, Y[:, 0]), grid, cvsearch.contiguous_folds(c1.n, c1.k),
                                     holdout=holdout)
    assert rep.method == "chol"
    assert rel(curve_of(rep, grid), g["exact_mean"][:, 0]) <= 1e-8
    assert int(np.argmin(curve_of(rep, grid))) == int(np.argmin(g["exact_mean"][:, 0]))


@pytest.mark.parametrize("batch", [32, 5, 1])
def test_exact_multi_output_batches(gpu, batch):
    # q = 17 in lambda batches of 32 / 5 (ragged last batch) / 1
    g = golden("small_multi_cv")
    grid = cvsearch.make_grid(float(g["lo"]), float(g["hi"]), int(g["q"]))
    n, k = g["X"].shape[0], int(g["k"])
    curves = exact.exact_curves(g["X"], g["Y"], [n // k] * k, grid.values, batch=batch)
    assert rel(curves.mean(axis=0), g["exact_mean"]) <= 1e-8


def test_exact_permuted_misclass_and_wide_outputs_vs_oracle(gpu):
    X, Y = configs.maclaurin(300, 24, m=2, seed=8)
    folds = cvsearch.make_folds(300, 3, seed=2)
    grid = cvsearch.make_grid(1e-3, 1e2, 9)
    ref = orc.grid_search_exact(X, Y, folds.assignments, 3, grid.values, metric=orc.MISCLASS)
    rep = cvsearch.grid_search_exact(cvsearch.Dataset(X, Y), grid, folds, metric=cvsearch.MISCLASS)
    assert np.array_equal(rep.curves, ref["curves"])
    # m = 20 outputs: two right-hand-side groups of the solve kernel
    X, Y = configs.powerlaw(250, 30, 20, seed=3)
    folds = cvsearch.make_folds(250, 5, seed=4)
    grid = cvsearch.make_grid(1e-3, 1e1, 7)
    ref = orc.grid_search_exact(X, Y, folds.assignments, 5, grid.values)
    rep = cvsearch.grid_search_exact(cvsearch.Dataset(X, Y), grid, folds)
    assert rel(rep.curves, ref["curves"]) <= 1e-8
    assert np.array_equal(rep.best_index, ref["best"])


def test_pichol_equals_exact_at_interpolating_samples(gpu):
    # g = r + 1: the polynomial interpolates the sampled factors, so the two sweeps agree there
    X, Y = configs.powerlaw(400, 40, 1, seed=5)
    grid = cvsearch.make_grid(1e-2, 1e1, 13)
    folds = cvsearch.contiguous_folds(400, 4)
    pi = cvsearch.grid_search_pichol(cvsearch.Dataset(X, Y), grid, folds, g=3, r=2)
    ex = cvsearch.grid_search_exact(cvsearch.Dataset(X, Y), grid, folds)
    for j in orc.sample_indices(13, 3):
        assert rel(pi.curves[:, j], ex.curves[:, j]) <= 1e-9


def test_exact_not_positive_definite(gpu):
    X = np.zeros((40, 6))
    X[:, 0] = 1.0
    Y = np.ones((40, 1))
    grid = cvsearch.make_grid(1e-3, 1.0, 5)
    with pytest.raises(NotPositiveDefinite):
        exact.exact_curves(X, Y, [10] * 4, -grid.values)


# ------------------------------------------------------------------ command line


def read_report(path):
    with open(path) as f:
        rows = list(csv.reader(f))
    return rows[0], [(r[0], int(r[1]), float(r[2]), float(r[3])) for r in rows[1:]]


@pytest.mark.parametrize("name", ["cv_pichol", "cv_chol", "cv_mis", "cv_mchol", "cv_pinrmse"])
def test_cli_cv_matches_reference(gpu, tmp_path, capsys, name):
    runs = json.load(open(os.path.join(GOLD, "runs.json")))
    argv = [os.path.join(GOLD, a) if a.endswith((".bin", ".csv")) else a for a in runs[name]["argv"]]
    out = str(tmp_path / "r.csv")
    assert cli.main(argv + ["--out", out, "--no-figures"]) == 0
    line = capsys.readouterr().out.strip()
    want = runs[name]["stdout"].split(", ")
    got = line.split(", ")
    assert got[:3] == want[:3]  # method, best lambda, best error (%.6g); wall seconds differ
    h_ref, ref = read_report(os.path.join(GOLD, name + ".csv"))
    h, rows = read_report(out)
    assert h == h_ref and len(rows) == len(ref)
    for a, b in zip(rows, ref):
        assert a[:3] == b[:3]
        assert abs(a[3] - b[3]) <= 1e-8 * max(abs(b[3]), 1e-300)


def test_cli_factor_path_matches_reference(gpu, tmp_path, capsys):
    runs = json.load(open(os.path.join(GOLD, "runs.json")))
    argv = [os.path.join(GOLD, a) if a.endswith(".bin") else a for a in runs["fp"]["argv"]]
    out = str(tmp_path / "fp.csv")
    assert cli.main(argv + ["--out", out, "--no-figures"]) == 0
    got = capsys.readouterr().out.strip().split(", ")
    want = runs["fp"]["stdout"].split(", ")
    assert got[:3] == want[:3]
    ref = np.loadtxt(os.path.join(GOLD, "fp.csv"), delimiter=",", skiprows=1)
    mine = np.loadtxt(out, delimiter=",", skiprows=1)
    assert np.array_equal(mine[:, [0, 2]], ref[:, [0, 2]])
    assert np.max(np.abs(mine[:, 1] - ref[:, 1])) <= 1e-8 * np.max(ref[:, 1])


def test_mchol_cost_formula_and_validation(gpu):
    # cvsearch.py:246-252: exactly 3 + 2 * ceil(log2(s0 / s_min)) factorizations per fold
    X, Y = configs.powerlaw(400, 30, 1, seed=2)
    folds = cvsearch.contiguous_folds(400, 4)
    rep = cvsearch.mchol_search(cvsearch.Dataset(X, Y[:, 0]), -1.5, 1.5, 0.0025, folds)
    assert rep.method == "mchol" and len(rep.per_lambda_error) == 3 + 2 * int(np.ceil(np.log2(1.5 / 0.0025)))
    assert rep.best_error == min(rep.per_lambda_error.values())
    with pytest.raises(UsageError):
        cvsearch.mchol_search(cvsearch.Dataset(X, Y[:, 0]), -1.5, 0.001, 0.01, folds)


def test_pinrmse_exact_at_samples_matches_oracle(gpu):
    # the sampled per-fold errors are exact hold-out errors (oracle.grid_search_exact at those lambdas)
    X, Y = configs.powerlaw(500, 40, 1, seed=4)
    folds = cvsearch.contiguous_folds(500, 5)
    grid = cvsearch.make_grid(1e-3, 1e1, 21)
    rep = cvsearch.pinrmse_search(cvsearch.Dataset(X, Y[:, 0]), grid, folds, g=5, r=2)
    sl = grid.values[orc.sample_indices(21, 5)]
    ref = orc.grid_search_exact(X, Y[:, 0], folds.assignments, 5, sl)
    assert rel(rep.curves, ref["curves"]) <= 1e-8
    assert rep.method == "pinrmse" and len(rep.per_lambda_error) == 21
