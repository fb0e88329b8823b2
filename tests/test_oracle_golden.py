"""Pin the CPU oracle (oracle/pichol_oracle.py) against fixtures produced by the REAL
reference package (tests/golden/make_golden.py imports /root/reference read-only).

These run without a GPU: they establish that the checker the CUDA path is compared
with reproduces the reference's own outputs on the same inputs.
"""

import numpy as np
import pytest

from oracle import pichol_oracle as orc
from paper_1404_0466_b200 import configs
from tests.conftest import golden


def test_c1_inputs_regenerate_identically():
    g = golden("c1_cv")
    X, Y = configs.generate(configs.CONFIGS["c1"])
    assert X.shape == (2000, 256) and Y.shape == (2000, 1)
    assert X.sum() == g["x_sum"] and Y.sum() == g["y_sum"]


def test_c1_full_sweep_matches_reference():
    g = golden("c1_cv")
    c1 = configs.CONFIGS["c1"]
    X, Y = configs.generate(c1)
    grid = orc.make_grid(c1.lo, c1.hi, c1.q)
    assert np.array_equal(grid, g["grid"])
    out = orc.grid_search_pichol(X, Y[:, 0], orc.contiguous_assignments(c1.n, c1.k), c1.k, grid, g=c1.s, r=c1.r)
    # multi-RHS composition vs the stock driver: same numbers up to summation order
    assert np.max(np.abs(out["curves"] - g["per_fold"]) / g["per_fold"]) <= 1e-12
    assert np.max(np.abs(out["mean"] - g["mean"]) / g["mean"]) <= 1e-12
    assert np.array_equal(out["best"], g["best"])
    assert grid[out["best"][0]] == g["best_lambda"][0]


def test_exact_search_matches_reference():  # cvsearch.grid_search_exact, cvsearch.py:178-203
    g = golden("c1_cv")
    c1 = configs.CONFIGS["c1"]
    X, Y = configs.generate(c1)
    grid = orc.make_grid(c1.lo, c1.hi, c1.q)
    out = orc.grid_search_exact(X, Y[:, 0], orc.contiguous_assignments(c1.n, c1.k), c1.k, grid)
    assert np.max(np.abs(out["mean"] - g["exact_mean"]) / g["exact_mean"]) <= 1e-12
    g = golden("small_multi_cv")
    grid = orc.make_grid(float(g["lo"]), float(g["hi"]), int(g["q"]))
    n, k = g["X"].shape[0], int(g["k"])
    out = orc.grid_search_exact(g["X"], g["Y"], orc.contiguous_assignments(n, k), k, grid)
    assert np.max(np.abs(out["mean"] - g["exact_mean"]) / g["exact_mean"]) <= 1e-12


@pytest.mark.parametrize("name", ["small_multi_cv", "small_misclass_cv"])
def test_small_cv_matches_reference(name):
    g = golden(name)
    grid = orc.make_grid(float(g["lo"]), float(g["hi"]), int(g["q"]))
    n, k = g["X"].shape[0], int(g["k"])
    out = orc.grid_search_pichol(g["X"], g["Y"], np.arange(n) // (n // k), k, grid, g=int(g["g"]), r=int(g["r"]),
                                 metric=str(g["metric"]))
    tol = 1e-12 if str(g["metric"]) == "rmse" else 0.0
    assert np.max(np.abs(out["curves"] - g["per_fold"])) <= tol * max(1.0, np.max(np.abs(g["per_fold"])))
    assert np.array_equal(out["best"], g["best"])


@pytest.mark.parametrize("kind,h0", [("recursive", 8), ("rowwise", 64), ("fullmatrix", 64)])
def test_fit_d40_matches_reference(kind, h0):
    g = golden("fit_d40")
    H = g["H"]
    if kind == "recursive":
        perm = orc.recursive_perm(40, h0)
    elif kind == "rowwise":
        perm = orc.rowwise_perm(40)
    else:
        perm = np.arange(40 * 40)
    mod = orc.fit(H, g["lams"], 2, perm=perm)
    theta = g[f"{kind}_theta"]
    assert np.max(np.abs(mod["theta"] - theta)) <= 1e-13 * np.max(np.abs(theta))
    assert abs(mod["residual_fro"] - float(g[f"{kind}_residual_fro"])) <= 1e-12
    assert mod["cond_V"] == float(g[f"{kind}_cond_V"])
    for j, lam in enumerate(g["eval_lams"]):
        assert np.max(np.abs(orc.eval_dense(mod, lam) - g[f"{kind}_L"][j])) <= 1e-13
        assert np.max(np.abs(orc.eval_vector(mod, lam) - g[f"{kind}_v"][j])) <= 1e-13


def test_solve_interp_matches_reference():
    g = golden("fit_d40")
    mod = orc.fit(g["H"], g["lams"], 2, perm=orc.recursive_perm(40, 8))
    for j, lam in enumerate(g["eval_lams"]):
        assert np.max(np.abs(orc.solve_interp(mod, g["g"], lam) - g["solve_theta"][j])) <= 1e-12
        assert np.max(np.abs(orc.solve_interp(mod, g["Gmat"], lam) - g["solve_multi"][j])) <= 1e-12
    for j, lam in enumerate(g["lams"]):
        assert np.max(np.abs(orc.cholesky(g["H"] + lam * np.eye(40)) - g["exact_L"][j])) <= 1e-14


def test_rescale_branch_matches_reference():
    g = golden("fit_rescale")
    mod = orc.fit(g["H"], g["lams"], 2)
    assert mod["cond_V"] > orc.COND_LIMIT
    assert mod["t_scale"] == float(g["t_scale"]) and mod["t_shift"] == float(g["t_shift"])
    assert np.max(np.abs(mod["theta"] - g["theta"])) <= 1e-9 * np.max(np.abs(g["theta"]))
    assert np.max(np.abs(orc.eval_dense(mod, g["lams"][2]) - g["L_mid"])) <= 1e-9


def test_wide_cubic_matches_reference():
    g = golden("fit_wide_cubic")
    mod = orc.fit(g["H"], g["lams"], 3, perm=orc.recursive_perm(24, 4))
    assert mod["t_scale"] == float(g["t_scale"]) and mod["t_shift"] == float(g["t_shift"])
    assert np.max(np.abs(mod["theta"] - g["theta"])) <= 1e-10 * np.max(np.abs(g["theta"]))
    for j, lam in enumerate(g["eval_lams"]):
        ref = g["L"][j]
        assert np.max(np.abs(orc.eval_dense(mod, lam) - ref)) <= 1e-10 * max(np.linalg.norm(ref), 1.0)


def test_layout_permutations_match_reference():
    g = golden("layouts")
    for key in g.files:
        parts = key.split("_")
        if parts[0] == "recursive":
            got = orc.recursive_perm(int(parts[1]), int(parts[2]))
        else:
            got = orc.rowwise_perm(int(parts[1]))
        assert np.array_equal(got, g[key]), key


def test_assemble_matches_reference():
    g = golden("assemble")
    H, G = orc.assemble(g["X"], g["Y"][:, 0])
    assert np.array_equal(H, g["H"])
    assert np.max(np.abs(G - g["g"])) <= 1e-13


def test_sample_indices_and_grid():
    assert orc.sample_indices(31, 4).tolist() == [0, 10, 20, 30]
    assert orc.sample_indices(200, 5).tolist() == [0, 50, 100, 149, 199]  # 99.5 -> 100 (half-to-even)
    assert orc.sample_indices(500, 6).tolist() == [0, 100, 200, 299, 399, 499]
    g = orc.make_grid(1e-4, 1e2, 200)
    assert g[0] == 1e-4 and g[-1] == 1e2


def test_oracle_error_kinds():
    with pytest.raises(orc.OracleError) as e:
        orc.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert e.value.kind == "NotPositiveDefinite"
    with pytest.raises(orc.OracleError) as e:
        orc.cholesky(np.array([[1.0, 0.5], [0.0, 1.0]]))
    assert e.value.kind == "NotSymmetric"
    with pytest.raises(orc.OracleError) as e:
        orc.fit(np.eye(3), [0.1, 0.2], 2)
    assert e.value.kind == "InsufficientSamples"
