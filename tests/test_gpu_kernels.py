"""Kernel-level parity of the CUDA path against the CPU oracle (oracle/pichol_oracle.py).

Every test calls through the C ABI (paper_1404_0466_b200._lib) and compares with
the oracle on the same seeded inputs. Tolerances: FP64 implementation noise
(different but valid summation orders) -- 1e-12 relative for Gram/Cholesky,
1e-10 * ||L||_F for interpolated factors (north_star), 1e-8 for hold-out errors.
"""

import numpy as np
import pytest

from oracle import pichol_oracle as orc
from paper_1404_0466_b200 import _dev, _lib, _ops, configs, pichol
from paper_1404_0466_b200.engine import PicholEngine
from tests.helpers import make_spd, make_spd_spectrum, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,m", [(300, 20, 2), (1000, 129, 3), (777, 256, 10), (2048, 300, 1)])
def test_gram_blocks_matches_numpy(gpu, n, d, m):
    X, Y = configs.powerlaw(n, d, m, seed=n + d)
    G, C = _ops.gram(X, Y)
    H = _dev.colmajor_to_host(G.reshape(-1), d)
    H_ref, C_ref = orc.assemble(X, Y)
    assert rel(H, H_ref) <= 1e-13
    assert np.array_equal(H, H.T)
    assert rel(C.cpu().numpy().T, C_ref) <= 1e-13


@pytest.mark.parametrize("d", [1, 2, 40, 127, 128, 129, 255, 300, 513])
def test_potrf_matches_lapack(gpu, d):
    rng = np.random.default_rng(d)
    A = make_spd(rng, d, shift=0.5)
    A = 0.5 * (A + A.T)
    dA = _dev.colmajor_to_dev(A).reshape(-1)
    info = _ops.potrf(dA, d, 1)
    assert info[0] == 0
    _ops.lower_of(dA, d)
    L = _dev.colmajor_to_host(dA, d)
    L_ref = orc.cholesky(A)
    assert np.max(np.abs(L - L_ref)) <= 1e-12 * np.linalg.norm(L_ref)
    assert np.linalg.norm(L @ L.T - A) <= 1e-13 * np.linalg.norm(A)


def test_potrf_batched_and_info(gpu):
    rng = np.random.default_rng(7)
    d = 200
    mats = [make_spd(rng, d) for _ in range(3)]
    bad = mats[1].copy()
    bad[150, 150] = -1e3  # leading minor of order 151 fails
    mats[1] = bad
    dA = _dev.to_dev(np.stack([np.ascontiguousarray(M.T) for M in mats]).reshape(3, -1))
    info = _ops.potrf(dA, d, 3)
    assert info[0] == 0 and info[2] == 0
    assert info[1] == 151
    for b in (0, 2):
        L = np.tril(dA[b].reshape(d, d).cpu().numpy().T)
        assert np.max(np.abs(L - orc.cholesky(mats[b]))) <= 1e-12 * np.linalg.norm(L)


@pytest.fixture
def chol_dmma():
    _lib.call("rp_set_option", b"chol_ozaki", 0)
    yield
    _lib.call("rp_set_option", b"chol_ozaki", 1)


@pytest.mark.parametrize("d", [1280, 1300, 2176])
@pytest.mark.parametrize("tensor", [True, False])
def test_potrf_trailing_update_paths(gpu, request, d, tensor):
    # d > 1024 runs trailing updates: on the int8 tensor cores (Ozaki) by default when
    # (d - 1024) % 128 == 0 (1280, 2176), FP64 DMMA otherwise (1300) or with the option off
    if not tensor:
        request.getfixturevalue("chol_dmma")
    mats = [make_spd_spectrum(d, 1e-3, 1e2, seed=d + b) for b in range(2)]
    mats = [0.5 * (M + M.T) for M in mats]
    dA = _dev.to_dev(np.stack([np.ascontiguousarray(M.T) for M in mats]).reshape(2, -1))
    info = _ops.potrf(dA, d, 2)
    assert list(info) == [0, 0]
    for b in range(2):
        L = np.tril(dA[b].reshape(d, d).cpu().numpy().T)
        L_ref = orc.cholesky(mats[b])
        assert np.linalg.norm(L - L_ref) <= 1e-12 * np.linalg.norm(L_ref)
        assert np.linalg.norm(L @ L.T - mats[b]) <= 1e-13 * np.linalg.norm(mats[b])


def test_potrf_batched_groups(gpu):
    # 9 matrices over the stream groups (ragged 3/2/2/2 split), a failure in the second group
    rng = np.random.default_rng(11)
    d = 300
    mats = [make_spd(rng, d) for _ in range(9)]
    mats[4] = mats[4].copy()
    mats[4][260, 260] = -1e3
    dA = _dev.to_dev(np.stack([np.ascontiguousarray(M.T) for M in mats]).reshape(9, -1))
    info = _ops.potrf(dA, d, 9)
    assert list(info) == [0, 0, 0, 0, 261, 0, 0, 0, 0]
    for b in (0, 3, 5, 8):
        L = np.tril(dA[b].reshape(d, d).cpu().numpy().T)
        assert np.max(np.abs(L - orc.cholesky(mats[b]))) <= 1e-12 * np.linalg.norm(L)


@pytest.mark.parametrize("d,r,s", [(40, 2, 4), (70, 1, 3), (130, 3, 6), (64, 2, 5)])
def test_fit_tiles_matches_oracle(gpu, d, r, s):
    H = make_spd_spectrum(d, 0.5, 50.0, seed=d)
    lams = np.logspace(-2, 1, s)
    lams_s, V, cond, ts, tsh, P = pichol.fit_basis(lams, r)
    mod = orc.fit(H, lams, r)
    assert cond == mod["cond_V"] and ts == mod["t_scale"] and tsh == mod["t_shift"]
    A = _dev.to_dev(np.stack([np.ascontiguousarray((H + l * np.eye(d)).T) for l in lams_s]).reshape(s, -1))
    info = _ops.potrf(A, d, s)
    assert np.all(info == 0)
    tiles, resid = _ops.fit_tiles(A, d, s, 1, r, P, V)
    theta = _ops.export_theta(tiles[0], d, r, orc.rowwise_perm(d), d * (d + 1) // 2)
    assert np.max(np.abs(theta - mod["theta"])) <= 1e-11 * np.max(np.abs(mod["theta"]))
    assert abs(float(resid.cpu()[0]) - mod["residual_fro"]) <= 1e-9 * max(mod["residual_fro"], 1e-12) + 1e-14
    for lam in (lams_s[0], 0.37, lams_s[-1]):
        t = ts * lam + tsh
        L = _ops.materialize(tiles[0], d, r, t)
        L_ref = orc.eval_dense(mod, lam)
        assert np.max(np.abs(L - L_ref)) <= 1e-10 * np.linalg.norm(L_ref)


@pytest.mark.parametrize("d,r,m,q", [(40, 2, 1, 7), (100, 2, 10, 31), (130, 3, 16, 5), (64, 1, 3, 40), (200, 2, 9, 18)])
def test_eval_solve_matches_oracle(gpu, d, r, m, q):
    H = make_spd_spectrum(d, 0.3, 30.0, seed=d + m)
    rng = np.random.default_rng(d * m)
    G = rng.standard_normal((d, m))
    grid = np.logspace(-2, 0, q)
    lams = np.logspace(-2, 0, r + 2)
    mod = orc.fit(H, lams, r)
    lams_s, V, cond, ts, tsh, P = pichol.fit_basis(lams, r)
    A = _dev.to_dev(np.stack([np.ascontiguousarray((H + l * np.eye(d)).T) for l in lams_s]).reshape(len(lams), -1))
    assert np.all(_ops.potrf(A, d, len(lams)) == 0)
    tiles, _ = _ops.fit_tiles(A, d, len(lams), 1, r, P, V)
    W, flags = _ops.eval_solve(tiles[0], d, r, G, ts * grid + tsh)
    assert not np.any(flags)
    for j, lam in enumerate(grid):
        ref = orc.solve_interp(mod, G, lam)
        assert rel(W[j], ref) <= 1e-10


def test_eval_solve_flags_singular(gpu):
    # indefinite H: the (0,0) entry sqrt(lam - 1/2) is fitted by a quadratic crossing zero
    H = np.diag([-0.5, 1.0])
    lams = np.linspace(1.0, 2.0, 4)
    mod = orc.fit(H, lams, 2)
    c0, c1, c2 = mod["theta"][:, 0]
    roots = [t.real for t in np.roots([c2, c1, c0]) if abs(t.imag) < 1e-9]
    lam_bad = next(l for l in sorted(roots) if 0 < l < 1.0)
    tiles = _ops.import_theta(mod["theta"], 2, 2, orc.rowwise_perm(2))
    _, flags = _ops.eval_solve(tiles, 2, 2, np.ones((2, 1)), [lam_bad, 1.5])
    assert flags[0] == 1 and flags[1] == 0


@pytest.mark.parametrize("metric", ["rmse", "misclass"])
def test_holdout_direct_matches_oracle(gpu, metric):
    rng = np.random.default_rng(3)
    nv, d, c = 517, 70, 12
    X = rng.standard_normal((nv, d))
    B = rng.standard_normal((d, c)) * 0.1
    Y = np.sign(rng.standard_normal((nv, c))) if metric == "misclass" else rng.standard_normal((nv, c))
    got = _ops.holdout(B, X, Y, metric)
    ref = orc.holdout_error(B, X, Y, metric)
    assert rel(got, ref) <= 1e-12


@pytest.mark.parametrize("holdout", ["direct", "gram"])
@pytest.mark.parametrize("n,d,m,k,q,s,r", [(600, 24, 3, 3, 17, 4, 2), (2000, 256, 1, 5, 31, 4, 2),
                                          (1500, 100, 10, 5, 20, 5, 2), (1200, 70, 16, 4, 9, 6, 3)])
def test_engine_sweep_matches_oracle(gpu, holdout, n, d, m, k, q, s, r):
    X, Y = configs.powerlaw(n, d, m, seed=n)
    assign = configs.contiguous_assignments(n, k)
    grid = orc.make_grid(1e-3, 1e1, q)
    ref = orc.grid_search_pichol(X, Y, assign, k, grid, g=s, r=r)
    lams_s, V, cond, ts, tsh, P = pichol.fit_basis(grid[orc.sample_indices(q, s)], r)
    eng = PicholEngine([n // k] * k, d, m, q, s, r, holdout=holdout)
    curves, mean, best = eng.sweep(_dev.to_dev(X), _dev.to_dev(Y), lams_s, P, V, ts * grid + tsh)
    assert eng.check_numerics(lams_s) is None
    assert rel(curves.cpu().numpy(), ref["curves"]) <= 1e-8
    assert rel(mean.cpu().numpy(), ref["mean"]) <= 1e-8
    assert np.array_equal(best.cpu().numpy(), ref["best"])


# ---------------------------------------------------------------- tensor-core (Ozaki) Gram


def normalized_err(G, G_ref):
    s = np.sqrt(np.outer(np.diag(G_ref), np.diag(G_ref)))
    s[s == 0] = 1.0
    return np.max(np.abs(np.tril(G) - np.tril(G_ref)) / s)


@pytest.mark.parametrize("n,d", [(1000, 256), (40000, 128), (3000, 384)])
def test_ozaki_gram_fp64_level(gpu, n, d):
    # per-column scales over 200 orders of magnitude; 40000 rows cut K into int32-safe chunks
    rng = np.random.default_rng(n + d)
    X = rng.standard_normal((n, d)) * np.logspace(-50, 50, d)
    G, _ = _ops.gram(X, None)
    G = _dev.colmajor_to_host(G.reshape(-1), d)
    G_ref = X.T @ X
    assert normalized_err(G, G_ref) <= 1e-14


@pytest.fixture
def gram_dmma():
    _lib.call("rp_set_option", b"gram_dmma", 1)
    yield
    _lib.call("rp_set_option", b"gram_dmma", 0)


def test_ozaki_gram_matches_dmma_gram(gpu, request):
    X, Y = configs.powerlaw(2500, 512, 3, seed=5)
    G1, C1 = _ops.gram(X, Y)
    request.getfixturevalue("gram_dmma")
    G2, C2 = _ops.gram(X, Y)
    G1 = _dev.colmajor_to_host(G1.reshape(-1), 512)
    G2 = _dev.colmajor_to_host(G2.reshape(-1), 512)
    err = normalized_err(G1, G2)
    assert err <= 1e-14, err
    assert np.array_equal(C1.cpu().numpy(), C2.cpu().numpy())  # X^T Y takes the same path


def test_ozaki_gram_zero_and_nonfinite_columns(gpu):
    rng = np.random.default_rng(9)
    X = rng.standard_normal((700, 256))
    X[:, 5] = 0.0
    X[123, 17] = np.nan
    X[9, 200] = np.inf
    G, _ = _ops.gram(X, None)
    G = _dev.colmajor_to_host(G.reshape(-1), 256)
    bad = np.zeros(256, bool)
    bad[[17, 200]] = True
    mask = bad[:, None] | bad[None, :]
    assert np.all(np.isnan(G[mask]))
    assert np.all(G[5, ~bad] == 0.0) and np.all(G[~bad, 5] == 0.0)
    keep = ~mask
    G_ref = np.nan_to_num(X).T @ np.nan_to_num(X)
    assert normalized_err(np.where(keep, G, 0.0), np.where(keep, G_ref, 0.0)) <= 1e-14


@pytest.fixture
def holdout_dmma():
    _lib.call("rp_set_option", b"holdout_ozaki", 0)
    yield
    _lib.call("rp_set_option", b"holdout_ozaki", 1)


@pytest.mark.parametrize("n,d,m,k,q", [(3000, 300, 3, 3, 45), (4000, 512, 10, 4, 13), (1500, 70, 1, 5, 9)])
def test_holdout_gram_tensor_core_matches_dmma(gpu, request, n, d, m, k, q):
    # the Gram-form hold-out on the int8 tensor cores (w^T T w from the lower triangle of G_f)
    # against the FP64 DMMA form and the oracle; d and q*m not multiples of the 128 tile
    X, Y = configs.powerlaw(n, d, m, seed=d + q)
    grid = orc.make_grid(1e-3, 1e1, q)
    lams_s, V, cond, ts, tsh, P = pichol.fit_basis(grid[orc.sample_indices(q, 4)], 2)
    eng = PicholEngine([n // k] * k, d, m, q, 4, 2, holdout="gram")
    c_tc = eng.sweep(_dev.to_dev(X), _dev.to_dev(Y), lams_s, P, V, ts * grid + tsh)[0].cpu().numpy()
    request.getfixturevalue("holdout_dmma")
    eng2 = PicholEngine([n // k] * k, d, m, q, 4, 2, holdout="gram")
    c_dm = eng2.sweep(_dev.to_dev(X), _dev.to_dev(Y), lams_s, P, V, ts * grid + tsh)[0].cpu().numpy()
    assert rel(c_tc, c_dm) <= 1e-10
    ref = orc.grid_search_pichol(X, Y, configs.contiguous_assignments(n, k), k, grid, g=4, r=2)
    assert rel(c_tc, ref["curves"]) <= 1e-8


@pytest.mark.parametrize("d", [130, 131, 256])
@pytest.mark.parametrize("nb", [3, 8, 11])
def test_fold_systems_fixed_order_sums(gpu, d, nb):
    """rp_fold_systems (row-pair kernel for even d, scalar kernel for odd d): A[f][s] = sum_{b != f} G_b +
    lam_s I over the lower triangle, bit-identical to the sequential sum in block order; nothing above the
    diagonal is read (NaN there) or written (sentinel kept); fold -1 holds nothing out."""
    torch = _dev.torch()
    rng = np.random.default_rng(d * 100 + nb)
    G = rng.standard_normal((nb, d, d))  # column-major blocks: G[b][j][i] = entry (i, j)
    low = np.triu(np.ones((d, d), dtype=bool))  # [j][i] with i >= j: the lower triangle of a column-major matrix
    G[:, ~low] = np.nan
    folds = np.array(list(range(min(nb, 4))) + [-1], dtype=np.int32)
    lams = np.array([0.25, 3.0, 1e-3])
    nf, s = len(folds), len(lams)
    sentinel = -7.25
    A = torch.full((nf, s, d, d), sentinel, dtype=torch.float64, device=_dev.device())
    dG = _dev.to_dev(G)
    _lib.call("rp_fold_systems", _lib.ptr(dG), None, nb, d, 0, _lib.host_ptr(folds), nf, _lib.host_ptr(lams), s,
              _lib.ptr(A), None, _lib.stream())
    Ah = A.cpu().numpy()
    for fi, f in enumerate(folds):
        ref = np.zeros((d, d))
        for b in range(nb):
            if b != f:
                ref = ref + np.where(low, G[b], 0.0)
        for si, lam in enumerate(lams):
            want = ref + lam * np.eye(d)
            got = Ah[fi, si]
            assert np.array_equal(got[low], want[low]), (f, si)
            assert np.all(got[~low] == sentinel), "entries above the diagonal written"
