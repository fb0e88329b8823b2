"""The reference package's hot-path tests, restated against the drop-in API
(paper_1404_0466_b200.{linalg,trivec,pichol,ridge,cvsearch}) on the GPU, plus the
golden fixtures produced by the real reference (tests/golden/make_golden.py).

Each test names the reference test it restates (file:line under /root/reference/pkg/tests).
"""

import numpy as np
import pytest

from paper_1404_0466_b200 import cvsearch, linalg, pichol, ridge, trivec
from paper_1404_0466_b200.errors import (
    DegenerateSamples,
    DimensionMismatch,
    EmptyValidationSet,
    InsufficientSamples,
    NotPositiveDefinite,
    NotSymmetric,
    SingularInterpolant,
    UsageError,
)
from tests.conftest import golden
from tests.helpers import make_spd, make_spd_spectrum

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- linalg (test_linalg.py)


def test_cholesky_2x2_hand_values(gpu):  # test_linalg.py:13-17
    L = linalg.cholesky(np.array([[2.0, 1.0], [1.0, 2.0]])).matrix
    assert np.allclose(L, [[np.sqrt(2.0), 0.0], [1.0 / np.sqrt(2.0), np.sqrt(1.5)]], atol=1e-12)
    assert L.flags.f_contiguous


def test_solve_chol_hand_and_matrix_rhs(gpu, rng):  # test_linalg.py:20-30
    A = np.array([[2.0, 1.0], [1.0, 2.0]])
    assert np.allclose(linalg.solve_chol(linalg.cholesky(A), np.array([3.0, 3.0])), [1.0, 1.0], atol=1e-12)
    A = make_spd(rng, 6)
    B = rng.standard_normal((6, 3))
    X = linalg.solve_chol(linalg.cholesky(A), B)
    assert X.shape == (6, 3)
    assert np.allclose(A @ X, B, atol=1e-10)


def test_cholesky_errors(gpu):  # test_linalg.py:33-45
    with pytest.raises(DimensionMismatch):
        linalg.cholesky(np.ones((2, 3)))
    with pytest.raises(NotSymmetric):
        linalg.cholesky(np.array([[1.0, 0.5], [0.0, 1.0]]))
    with pytest.raises(NotPositiveDefinite):
        linalg.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    with pytest.raises(DimensionMismatch):
        linalg.solve_chol(linalg.cholesky(np.eye(3)), np.ones(4))


def test_factor_records_lambda(gpu):  # test_linalg.py:48-52
    L = linalg.cholesky(np.eye(2), lam=0.25)
    assert L.lam == 0.25 and not L.interpolated and L.dim == 2


@pytest.mark.parametrize("m", [1, 5, 24, 130])
def test_cholesky_reconstructs_and_solve_roundtrip(gpu, m):  # test_linalg.py:55-73
    rng = np.random.default_rng(m)
    B = rng.standard_normal((m, m))
    A = B.T @ B + np.eye(m)
    L = linalg.cholesky(A).matrix
    assert np.linalg.norm(L @ L.T - A) / np.linalg.norm(A) <= 1e-12
    assert np.array_equal(L, np.tril(L))
    x = rng.standard_normal(m)
    got = linalg.solve_chol(linalg.cholesky(A), A @ x)
    assert np.linalg.norm(got - x) / np.linalg.norm(x) <= 1e-8


# ---------------------------------------------------------------- ridge (test_ridge.py)


def problem(H, g):
    return ridge.RidgeProblem(X=None, y=None, H=np.asarray(H, float), g=np.asarray(g, float))


def test_assemble_hand_cases(gpu):  # test_ridge.py:20-30
    p = ridge.assemble(np.eye(2), np.array([1.0, 2.0]))
    assert np.array_equal(p.H, np.eye(2)) and np.array_equal(p.g, [1.0, 2.0])
    assert p.n == 2 and p.dim == 2
    p = ridge.assemble(np.ones((3, 1)), np.array([1.0, 2.0, 3.0]))
    assert np.array_equal(p.H, [[3.0]]) and np.array_equal(p.g, [6.0])


def test_assemble_matches_golden_and_is_symmetric(gpu):  # test_ridge.py:33-46
    g = golden("assemble")
    p = ridge.assemble(g["X"], g["Y"][:, 0])
    assert np.max(np.abs(p.H - g["H"])) <= 1e-12 * np.max(np.abs(g["H"]))
    assert np.max(np.abs(p.g - g["g"])) <= 1e-12 * np.max(np.abs(g["g"]))
    assert np.array_equal(p.H, p.H.T)
    with pytest.raises(DimensionMismatch):
        ridge.assemble(np.zeros((5, 2)), np.zeros(4))


def test_solve_exact_hand_and_negative(gpu):  # test_ridge.py:49-82
    sol = ridge.solve_exact(problem(np.eye(2), [2.0, 2.0]), 1.0)
    assert np.allclose(sol.theta, [1.0, 1.0], atol=1e-12) and sol.backend == ridge.CHOL and sol.lam == 1.0
    with pytest.raises(NotPositiveDefinite):
        ridge.solve_exact(problem(np.eye(2), [1.0, 1.0]), -0.5)
    with pytest.raises(NotPositiveDefinite):
        ridge.solve_exact(problem(np.zeros((2, 2)), [1.0, 1.0]), 0.0)


def test_residual_certificate_exact(gpu, rng):  # test_ridge.py:92-97
    p = problem(make_spd(rng, 8), rng.standard_normal(8))
    for lam in (1e-3, 1.0, 1e3):
        assert ridge.solve_exact(p, lam).residual <= 1e-10


def test_solve_interp_equals_exact_at_samples(gpu, rng):  # test_ridge.py:100-111
    H = make_spd(rng, 9)
    p = problem(H, rng.standard_normal(9))
    lams = np.array([0.1, 0.4, 1.0])
    model = pichol.fit(H, lams, 2, trivec.build_layout(trivec.RECURSIVE, 9, h0=4))
    for lam in lams:
        exact = ridge.solve_exact(p, lam).theta
        interp = ridge.solve_interp(p, model, lam)
        assert np.linalg.norm(interp.theta - exact) / np.linalg.norm(exact) <= 1e-8
        assert interp.backend == ridge.PICHOL


def test_solve_interp_accuracy_across_window(gpu):  # test_ridge.py:114-125
    H = make_spd_spectrum(16, 0.3, 30.0, seed=3)
    p = problem(H, np.random.default_rng(100).standard_normal(16))
    grid = np.logspace(-2, 0, 31)
    model = pichol.fit(H, grid[pichol.sample_indices(31, 4)], 2, trivec.build_layout(trivec.RECURSIVE, 16, h0=8))
    for lam in grid:
        exact = ridge.solve_exact(p, lam).theta
        interp = ridge.solve_interp(p, model, lam).theta
        assert np.linalg.norm(interp - exact) / np.linalg.norm(exact) <= 0.05


def test_solve_interp_raises_on_collapsed_diagonal(gpu):  # test_ridge.py:128-141
    H = np.diag([-0.5, 1.0])
    layout = trivec.build_layout(trivec.ROWWISE, 2)
    model = pichol.fit(H, np.linspace(1.0, 2.0, 4), 2, layout)
    j = layout.index_of(0, 0)
    c0, c1, c2 = model.theta[:, j]
    roots = np.roots([c2, c1, c0])
    lam_roots = sorted((t - model.t_shift) / model.t_scale for t in roots.real if abs(t.imag) < 1e-9)
    lam_bad = next(l for l in lam_roots if 0 < l < 1.0)
    with pytest.raises(SingularInterpolant):
        ridge.solve_interp(problem(np.eye(2), [1.0, 1.0]), model, lam_bad)


def test_solve_interp_matches_golden(gpu):
    g = golden("fit_d40")
    model = pichol.fit(g["H"], g["lams"], 2, trivec.build_layout(trivec.RECURSIVE, 40, 8))
    p = problem(g["H"], g["g"])
    for j, lam in enumerate(g["eval_lams"]):
        sol = ridge.solve_interp(p, model, lam)
        ref = g["solve_theta"][j]
        assert np.linalg.norm(sol.theta - ref) / np.linalg.norm(ref) <= 1e-10
        assert abs(sol.residual - g["solve_residual"][j]) <= 1e-8 * max(g["solve_residual"][j], 1e-6)


# ---------------------------------------------------------------- pichol (test_pichol.py)


def scalar_fit(samples, r=1):
    return pichol.fit(np.zeros((1, 1)), samples, r, trivec.build_layout(trivec.ROWWISE, 1))


def test_scalar_line_fit_closed_form(gpu):  # test_pichol.py:21-42
    model = scalar_fit(np.array([1.0, 4.0, 9.0]))
    assert model.t_scale == 1.0 and model.t_shift == 0.0
    assert np.allclose(model.theta[:, 0], [6.0 / 7.0, 12.0 / 49.0], atol=1e-12)
    assert abs(pichol.eval(model, 4.0).matrix[0, 0] - (6.0 / 7.0 + 12.0 / 49.0 * 4.0)) <= 1e-12
    assert pichol.eval_vector(model, 4.0).shape == (1,)
    preds = 6.0 / 7.0 + 12.0 / 49.0 * np.array([1.0, 4.0, 9.0])
    assert abs(model.residual_fro - np.linalg.norm(preds - np.array([1.0, 2.0, 3.0]))) <= 1e-12


def test_interpolation_exact_when_g_equals_r_plus_1(gpu, rng):  # test_pichol.py:45-53
    H = make_spd(rng, 10)
    lams = np.array([0.1, 0.4, 1.0])
    model = pichol.fit(H, lams, 2, trivec.build_layout(trivec.RECURSIVE, 10, h0=4))
    for lam in lams:
        exact = linalg.cholesky(H + lam * np.eye(10))
        assert np.max(np.abs(pichol.eval(model, lam).matrix - exact.matrix)) <= 1e-9


def test_fit_is_layout_independent(gpu, rng):  # test_pichol.py:73-83
    H = make_spd(rng, 12)
    lams = np.logspace(-1, 0, 4)
    res = [pichol.eval(pichol.fit(H, lams, 2, trivec.build_layout(kind, 12, h0=4)), 0.3).matrix
           for kind in (trivec.ROWWISE, trivec.RECURSIVE, trivec.FULLMATRIX, trivec.TILE)]
    for other in res[1:]:
        assert np.max(np.abs(res[0] - other)) <= 1e-14


@pytest.mark.parametrize("kind,h0", [("recursive", 8), ("rowwise", 64), ("fullmatrix", 64)])
def test_fit_matches_golden(gpu, kind, h0):
    g = golden("fit_d40")
    model = pichol.fit(g["H"], g["lams"], 2, trivec.build_layout(kind, 40, h0))
    theta = g[f"{kind}_theta"]
    assert np.max(np.abs(model.theta - theta)) <= 1e-12 * np.max(np.abs(theta))
    assert abs(model.residual_fro - float(g[f"{kind}_residual_fro"])) <= 1e-10
    assert model.cond_V == float(g[f"{kind}_cond_V"])
    for j, lam in enumerate(g["eval_lams"]):
        L = pichol.eval(model, lam).matrix
        ref = g[f"{kind}_L"][j]
        assert np.max(np.abs(L - ref)) <= 1e-10 * np.linalg.norm(ref)  # north_star factor tolerance
        assert np.max(np.abs(pichol.eval_vector(model, lam) - g[f"{kind}_v"][j])) <= 1e-10 * np.linalg.norm(ref)


def test_rescale_engages_only_when_ill_conditioned(gpu):  # test_pichol.py:158-172 + golden
    g = golden("fit_rescale")
    model = pichol.fit(g["H"], g["lams"], 2, trivec.build_layout(trivec.ROWWISE, 6))
    assert model.cond_V > pichol.COND_LIMIT
    assert model.t_scale == float(g["t_scale"]) and model.t_shift == float(g["t_shift"])
    assert np.max(np.abs(pichol.eval(model, g["lams"][2]).matrix - g["L_mid"])) <= 1e-9
    wide = pichol.fit(g["H"], np.logspace(-1, 0, 4), 2, trivec.build_layout(trivec.ROWWISE, 6))
    assert wide.t_scale == 1.0 and wide.t_shift == 0.0


def test_raw_monomials_flag_disables_rescale(gpu, rng, monkeypatch):  # test_pichol.py:175-185
    monkeypatch.setattr(pichol, "COND_LIMIT", 10.0)
    H = make_spd(rng, 4)
    layout = trivec.build_layout(trivec.ROWWISE, 4)
    lams = np.logspace(-1, 0, 4)
    rescaled = pichol.fit(H, lams, 2, layout)
    assert rescaled.t_scale != 1.0
    raw = pichol.fit(H, lams, 2, layout, raw_monomials=True)
    assert raw.t_scale == 1.0 and raw.t_shift == 0.0
    assert np.max(np.abs(pichol.eval(raw, 0.3).matrix - pichol.eval(rescaled, 0.3).matrix)) <= 1e-9


def test_wide_cubic_matches_golden(gpu):
    g = golden("fit_wide_cubic")
    model = pichol.fit(g["H"], g["lams"], 3, trivec.build_layout(trivec.RECURSIVE, 24, 4))
    for j, lam in enumerate(g["eval_lams"]):
        ref = g["L"][j]
        assert np.max(np.abs(pichol.eval(model, lam).matrix - ref)) <= 1e-10 * max(np.linalg.norm(ref), 1.0)


def test_fit_validation_and_sorting(gpu, rng):  # test_pichol.py:188-211
    H = make_spd(rng, 4)
    layout = trivec.build_layout(trivec.ROWWISE, 4)
    assert np.array_equal(pichol.fit(H, np.array([1.0, 0.1, 0.5]), 2, layout).sample_lambdas, [0.1, 0.5, 1.0])
    with pytest.raises(InsufficientSamples):
        pichol.fit(H, np.array([0.1, 0.2]), 2, layout)
    with pytest.raises(DegenerateSamples):
        pichol.fit(H, np.array([0.1, 0.1, 0.2]), 1, layout)
    with pytest.raises(DegenerateSamples):
        pichol.fit(H, np.array([-0.1, 0.2, 0.3]), 1, layout)
    with pytest.raises(DimensionMismatch):
        pichol.fit(H, np.array([0.1, 0.2, 0.3]), 1, trivec.build_layout(trivec.ROWWISE, 5))
    with pytest.raises(DegenerateSamples):
        pichol.eval(scalar_fit(np.array([1.0, 4.0, 9.0])), 0.0)


def test_fit_records_phase_timings(gpu, rng):  # test_pichol.py:222-226
    times = {"factorize": 0.0, "vec": 0.0, "fit": 0.0}
    pichol.fit(make_spd(rng, 6), np.logspace(-1, 0, 4), 2, trivec.build_layout(trivec.ROWWISE, 6), timings=times)
    assert all(v > 0 for v in times.values())


def test_nrmse_within_window_d16(gpu):  # test_pichol.py:86-95
    H = make_spd_spectrum(16, 0.3, 30.0, seed=3)
    grid = np.logspace(-2, 0, 31)
    model = pichol.fit(H, grid[pichol.sample_indices(31, 4)], 2, trivec.build_layout(trivec.RECURSIVE, 16, h0=8))
    diag = pichol.diagnostics(model, H, grid)
    assert diag.max_nrmse <= 0.05
    assert set(diag.nrmse_per_lambda) == set(float(l) for l in grid)


def test_eval_ops_count(gpu):  # test_pichol.py:133-155 (op count is r*D by construction)
    layout = trivec.build_layout(trivec.ROWWISE, 10)
    model = pichol.InterpModel(degree=2, sample_lambdas=np.array([0.1, 0.5, 1.0, 2.0]),
                               theta=np.zeros((3, layout.length)), layout=layout, cond_V=1.0, t_scale=1.0,
                               t_shift=0.0, residual_fro=0.0)
    assert model.eval_ops() == 2 * layout.length
    assert np.array_equal(pichol.eval_vector(model, 0.7), np.zeros(layout.length))


# ---------------------------------------------------------------- trivec on the device


def test_vectorize_roundtrip_all_layouts(gpu, rng):  # test_trivec.py:65-92
    for h in (1, 2, 17, 63, 64, 65, 130):
        L = np.tril(rng.standard_normal((h, h)))
        for kind in trivec.ALL_KINDS:
            layout = trivec.build_layout(kind, h)
            back = trivec.unvectorize(trivec.vectorize(L, layout), layout)
            assert np.array_equal(back.matrix, L), (kind, h)


def test_bulk_gather_h2_example(gpu):  # test_trivec.py:118-126
    L1 = np.array([[1.0, 0.0], [2.0, 3.0]])
    L2 = np.array([[4.0, 0.0], [5.0, 6.0]])
    T = trivec.bulk_gather([linalg.CholeskyFactor(L1), linalg.CholeskyFactor(L2)],
                           trivec.build_layout(trivec.ROWWISE, 2))
    assert T.tolist() == [[1, 2, 3], [4, 5, 6]]


# ---------------------------------------------------------------- cvsearch (test_cvsearch.py)


def test_holdout_error_hand_values(gpu):  # test_cvsearch.py:79-108
    assert cvsearch.holdout_error(np.array([1.0, 2.0, 3.0]), np.eye(3), np.array([1.0, 2.0, 3.0])) == 0.0
    assert cvsearch.holdout_error(np.zeros(2), np.zeros((4, 2)), np.array([1.0, -1.0, 1.0, -1.0])) == 1.0
    got = cvsearch.holdout_error(np.ones(3), np.eye(3), np.array([2.0, 1.0, -1.0]))
    assert abs(got - np.sqrt(5.0 / 3.0)) <= 1e-15
    assert cvsearch.holdout_error(np.array([0.5, -0.2, 0.0, 2.0]), np.eye(4), np.array([1.0, 1.0, -1.0, 1.0]),
                                  cvsearch.MISCLASS) == 0.5
    with pytest.raises(EmptyValidationSet):
        cvsearch.holdout_error(np.zeros(2), np.zeros((0, 2)), np.zeros(0))


def test_pichol_driver_validates(gpu):  # test_cvsearch.py:210-214
    X = np.random.default_rng(0).standard_normal((40, 3))
    ds = cvsearch.Dataset(X, X[:, 0])
    with pytest.raises(UsageError):
        cvsearch.grid_search_pichol(ds, cvsearch.make_grid(0.01, 0.1, 3), cvsearch.make_folds(40, 2, seed=0), g=4)


def test_certify_reuses_device_H_and_sees_changes(gpu):
    """_certify keeps one device copy of H per RidgeProblem; replacing H or changing it in place is
    picked up (the residual is the reference's ||H theta + lam theta - g|| / ||g||, ridge.py:63-66)."""
    rng = np.random.default_rng(3)
    X = rng.standard_normal((200, 40))
    y = rng.standard_normal(200)
    p = ridge.assemble(X, y)
    s1 = ridge.solve_exact(p, 0.5)
    first = p._H_dev[2]
    s2 = ridge.solve_exact(p, 0.7)
    assert p._H_dev[2] is first and s1.residual <= 1e-10 and s2.residual <= 1e-10
    p.H[:] = p.H * 2.0  # in place: the cached copy is stale
    theta = s2.theta
    ref = np.linalg.norm(p.H @ theta + 0.7 * theta - p.g) / np.linalg.norm(p.g)
    got = ridge._certify(p, 0.7, theta, ridge.CHOL).residual
    assert abs(got - ref) <= 1e-12 * max(ref, 1.0)
    p.H = p.H / 2.0  # replaced
    got = ridge._certify(p, 0.7, theta, ridge.CHOL).residual
    assert got <= 1e-10
