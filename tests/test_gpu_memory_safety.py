"""Out-of-bounds writes and races, without compute-sanitizer (closed on this GPU pool).

* Red zones: every output and workspace buffer of a C-ABI call sits inside a larger allocation whose
  margins hold a sentinel pattern; the call must leave the margins -- and the padding columns / padding
  between batched matrices inside the buffers -- untouched. This catches stray global stores of the
  bulk-copy / TMA-fed kernels (Ozaki SYRK, warp-specialised GEMM, fused eval+solve, fit).
* Races: the fused eval+solve's chunks, rings and chunk-private rows must not change results. Every
  lambda's arithmetic is independent of the chunk it runs in, so every chunking (each specialised chunk
  size and the generic kernel) must give bit-identical solutions; whole sweeps repeated on the same data
  must give bit-identical curves.
"""

import numpy as np
import pytest

from oracle import pichol_oracle as orc
from paper_1404_0466_b200 import _dev, _lib, _ops, configs, pichol
from paper_1404_0466_b200._lib import call, ptr, stream
from paper_1404_0466_b200.engine import PicholEngine, padded, tile_elems
from tests.helpers import make_spd_spectrum, rel

pytestmark = pytest.mark.gpu

SENTINEL = np.int64(0x7FF8DEADBEEF5A5A)  # a NaN payload no kernel writes
MARGIN = 8192  # doubles (64 KB, keeps 1 KB alignment of the interior)


class Guarded:
    """A device buffer of `n` doubles (or bytes, as doubles) between two sentinel margins."""

    def __init__(self, n, dtype=None):
        torch = _dev.torch()
        self.n = int(n)
        self.raw = torch.full((self.n + 2 * MARGIN,), int(SENTINEL), dtype=torch.int64, device=_dev.device())
        self.f64 = self.raw.view(torch.float64)
        self.buf = self.f64[MARGIN:MARGIN + self.n]

    def fill_(self, value):
        self.buf.fill_(value)
        return self

    def margins_intact(self):
        torch = _dev.torch()
        torch.cuda.synchronize()
        lo = self.raw[:MARGIN].cpu().numpy()
        hi = self.raw[MARGIN + self.n:].cpu().numpy()
        return bool(np.all(lo == SENTINEL) and np.all(hi == SENTINEL))


def guarded_ws(nbytes):
    return Guarded((int(nbytes) + 7) // 8 + 1)


def test_gram_blocks_stay_in_bounds(gpu):
    """Tensor-core (Ozaki, d % 128 == 0) and DMMA Gram blocks write only their d x d lower tiles, C and the
    workspace."""
    n_blk, d, m, nb = 700, 256, 3, 3
    rng = np.random.default_rng(5)
    X = rng.standard_normal((n_blk * nb, d))
    Y = rng.standard_normal((n_blk * nb, m))
    dX, dY = _dev.to_dev(X), _dev.to_dev(Y)
    for dmma in (0, 1):
        call("rp_set_option", b"gram_dmma", dmma)
        try:
            G = Guarded(nb * d * d).fill_(0.0)
            C = Guarded(nb * d * m).fill_(0.0)
            ws = guarded_ws(_lib.query("rp_gram_workspace_size", d, n_blk, nb))
            call("rp_gram_blocks", ptr(dX), d, n_blk, nb, d, ptr(dY), m, m, ptr(G.buf), ptr(C.buf), ptr(ws.buf),
                 stream())
            assert G.margins_intact() and C.margins_intact() and ws.margins_intact(), f"gram_dmma={dmma}"
            Gh = G.buf.cpu().numpy().reshape(nb, d, d)
            for b in range(nb):
                Xb = X[b * n_blk:(b + 1) * n_blk]
                ref = Xb.T @ Xb
                low = np.tril(Gh[b].T)  # column-major: G[b][j][i] = G(i, j); lower tiles written
                assert rel(low, np.tril(ref)) <= 1e-13
        finally:
            call("rp_set_option", b"gram_dmma", 0)


@pytest.mark.parametrize("chol_ozaki", [1, 0])
def test_potrf_leaves_batch_padding_alone(gpu, chol_ozaki):
    """Batched Cholesky with a matrix stride larger than d*d: the gaps between matrices, the info vector's
    neighbours and the workspace margins keep their sentinels."""
    d, batch, gap = 1024, 3, 5000
    stride = d * d + gap
    A = Guarded(batch * stride)
    mats = [make_spd_spectrum(d, 0.5, 40.0, seed=7 + b) for b in range(batch)]
    for b, M in enumerate(mats):
        A.buf[b * stride:b * stride + d * d].copy_(_dev.to_dev(np.ascontiguousarray(M.T).reshape(-1)))
    torch = _dev.torch()
    info_raw = torch.full((batch + 64,), -12345, dtype=torch.int32, device=_dev.device())
    info = info_raw[32:32 + batch]
    ws = guarded_ws(_lib.query("rp_potrf_workspace_size", d, batch))
    call("rp_set_option", b"chol_ozaki", chol_ozaki)
    try:
        call("rp_potrf_batched", ptr(A.buf), d, stride, batch, ptr(info), ptr(ws.buf), stream())
    finally:
        call("rp_set_option", b"chol_ozaki", 1)
    assert A.margins_intact() and ws.margins_intact()
    ih = info_raw.cpu().numpy()
    assert np.all(ih[:32] == -12345) and np.all(ih[32 + batch:] == -12345) and np.all(ih[32:32 + batch] == 0)
    raw = A.raw[MARGIN:MARGIN + batch * stride].cpu().numpy()
    for b in range(batch):
        assert np.all(raw[b * stride + d * d:(b + 1) * stride] == SENTINEL), f"gap after matrix {b} written"
        L = np.tril(A.buf[b * stride:b * stride + d * d].cpu().numpy().reshape(d, d).T)
        ref = np.linalg.cholesky(mats[b])
        assert np.linalg.norm(L - ref) <= 1e-12 * np.linalg.norm(ref)


def test_fit_tiles_stays_in_bounds(gpu):
    d, s, r, nf = 200, 4, 2, 2
    lams = np.logspace(-2, 0, s)
    mats = [make_spd_spectrum(d, 0.3, 30.0, seed=11 + f) for f in range(nf)]
    A = _dev.to_dev(np.stack([np.ascontiguousarray((M + l * np.eye(d)).T).reshape(-1)
                              for M in mats for l in lams]).reshape(-1))
    assert np.all(_ops.potrf(A, d, nf * s) == 0)
    _, V, _, _, _, Pm = pichol.fit_basis(lams, r)
    theta = Guarded(nf * tile_elems(d, r + 1)).fill_(0.0)
    resid = Guarded(nf).fill_(0.0)
    ws = guarded_ws(_lib.query("rp_fit_workspace_size", d, nf, s, r))
    Pm = np.ascontiguousarray(Pm, dtype=np.float64)
    Vm = np.ascontiguousarray(V, dtype=np.float64)
    call("rp_fit_tiles", ptr(A), d, s, nf, r, _lib.host_ptr(Pm), _lib.host_ptr(Vm), ptr(theta.buf), ptr(resid.buf),
         ptr(ws.buf), stream())
    assert theta.margins_intact() and resid.margins_intact() and ws.margins_intact()
    assert np.all(np.isfinite(theta.buf.cpu().numpy()))


def _solve_setup(d, r, m, seed):
    H = make_spd_spectrum(d, 0.3, 30.0, seed=seed)
    lams = np.logspace(-2, 0, r + 3)
    lams_s, V, _, ts, tsh, Pm = pichol.fit_basis(lams, r)
    A = _dev.to_dev(np.stack([np.ascontiguousarray((H + l * np.eye(d)).T) for l in lams_s]).reshape(len(lams), -1))
    assert np.all(_ops.potrf(A, d, len(lams)) == 0)
    tiles, _ = _ops.fit_tiles(A, d, len(lams), 1, r, Pm, V)
    G = np.random.default_rng(seed).standard_normal((d, m))
    return H, lams, tiles, G, ts, tsh


def _guarded_solve(tiles, d, r, G, tv, pad_cols=6):
    """rp_eval_solve with W (ldw padding columns), flags and workspace inside red zones."""
    torch = _dev.torch()
    m = G.shape[1]
    q = tv.shape[0]
    dp = padded(d)
    R = _dev.zeros((dp, m))
    R[:d].copy_(torch.from_numpy(np.ascontiguousarray(G)))
    ldw = q * m + pad_cols + ((q * m + pad_cols) & 1)
    W = Guarded(dp * ldw)
    fl_raw = torch.full((q + 64,), -777, dtype=torch.int32, device=_dev.device())
    fl = fl_raw[32:32 + q]
    ws = guarded_ws(_lib.query("rp_eval_solve_workspace_size", d, r, 1, m, q))
    call("rp_eval_solve", ptr(tiles), d, r, 1, ptr(R), m, ptr(_dev.to_dev(tv)), q, ptr(W.buf), ldw, ptr(fl), ptr(ws.buf),
         stream())
    assert W.margins_intact() and ws.margins_intact()
    flh = fl_raw.cpu().numpy()
    assert np.all(flh[:32] == -777) and np.all(flh[32 + q:] == -777)
    Wr = W.raw[MARGIN:MARGIN + dp * ldw].cpu().numpy().reshape(dp, ldw)
    assert np.all(Wr[:, q * m:] == SENTINEL), "padding columns of W written"
    Wh = W.buf.cpu().numpy().reshape(dp, ldw)[:d, :q * m].reshape(d, q, m).transpose(1, 0, 2)
    return Wh, flh[32:32 + q]


@pytest.fixture
def solve_lam():
    yield lambda v: call("rp_set_option", b"solve_lam", v)
    call("rp_set_option", b"solve_lam", 0)


@pytest.mark.parametrize("m,r,lams", [(10, 2, [2, 3, 4, 6, 8, 9, 10, 11, 12, 16]), (1, 2, [8, 16]), (16, 3, [4, 6, 7, 8])])
def test_eval_solve_bit_identical_across_chunkings(gpu, solve_lam, m, r, lams):
    """Every specialised chunk size and the planner's choice give bit-identical W (a race between chunks,
    ring stages or chunk-private rows would show up as a difference); the result matches the oracle; and
    no call writes outside W's q*m columns, the flags or the workspace."""
    d, q = 330, 37 if m % 2 == 0 else 38
    H, lams_s, tiles, G, ts, tsh = _solve_setup(d, r, m, seed=3 + m)
    grid = np.logspace(-2, 0, q)
    tv = ts * grid + tsh
    base, flags = _guarded_solve(tiles, d, r, G, tv)
    assert not np.any(flags)
    mod = orc.fit(H, lams_s, r)
    assert max(rel(base[j], orc.solve_interp(mod, G, l)) for j, l in enumerate(grid)) <= 1e-10
    for lam in lams:
        solve_lam(lam)
        W, _ = _guarded_solve(tiles, d, r, G, tv)
        assert np.array_equal(W, base), f"chunk {lam}: solutions differ from the planner's chunking"
    solve_lam(0)
    for _ in range(2):
        W, _ = _guarded_solve(tiles, d, r, G, tv)
        assert np.array_equal(W, base)


@pytest.mark.parametrize("nf,q", [(8, 200), (8, 196), (5, 103)])
def test_eval_solve_split_plan_bit_identical(gpu, solve_lam, nf, q):
    """One wave of CTAs that leaves SMs idle (8 folds x 17 chunks of 12 lambdas on 148 SMs) is planned as
    a main launch of smaller chunks plus a tail launch for each fold's last lambdas on the idle SMs (a tail
    CTA runs several folds' tails in turn). The solutions are bit-identical to single-launch chunkings,
    match the oracle, and W, flags and the workspace (main + tail rows) stay inside their red zones."""
    m, r, d = 10, 2, 200
    H, lams_s, tiles1, G, ts, tsh = _solve_setup(d, r, m, seed=77)
    torch = _dev.torch()
    te = tile_elems(d, r + 1)
    tiles = _dev.empty((nf * te,))
    for f in range(nf):
        tiles[f * te:(f + 1) * te].copy_(tiles1.reshape(-1)[:te] * (1.0 + f))
    grid = np.logspace(-2, 0, q)
    tv = ts * grid + tsh
    dp = padded(d)
    rhs = _dev.zeros((nf, dp, m))
    rhs[:, :d].copy_(torch.from_numpy(np.ascontiguousarray(G)).unsqueeze(0))
    ldw = q * m + 4

    def run():
        W = Guarded(nf * dp * ldw)
        fl = Guarded(nf * q)
        ws = guarded_ws(_lib.query("rp_eval_solve_workspace_size", d, r, nf, m, q))
        call("rp_eval_solve", ptr(tiles), d, r, nf, ptr(rhs), m, ptr(_dev.to_dev(tv)), q, ptr(W.buf), ldw,
             ptr(fl.buf), ptr(ws.buf), stream())
        assert W.margins_intact() and fl.margins_intact() and ws.margins_intact()
        assert not np.any(fl.raw[MARGIN:MARGIN + fl.n].view(torch.int32)[:nf * q].cpu().numpy())
        Wi = W.raw[MARGIN:MARGIN + nf * dp * ldw].cpu().numpy().reshape(nf, dp, ldw)
        assert np.all(Wi[:, :, q * m:] == SENTINEL), "padding columns of W written"
        return W.buf.cpu().numpy().reshape(nf, dp, ldw)[:, :d, :q * m].copy()

    solve_lam(0)
    plan = np.zeros(4, dtype=np.int32)
    call("rp_eval_solve_plan", d, r, nf, m, q, _lib.host_ptr(plan))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    assert plan[0] >= 1 and plan[0] * plan[1] + plan[2] >= q  # main chunks + tail cover the grid
    if plan[2]:  # split plan: main CTAs + tail CTAs fit the device together
        assert nf * plan[1] + plan[3] <= sms and 1 <= plan[3] <= nf
    if (nf, q, sms) == (8, 200, 148):
        assert tuple(plan) == (11, 18, 2, 4), plan
    base = run()  # the planner's choice (the split plan at (8, 200) on a 148-SM device)
    mod = orc.fit(H, lams_s, r)
    for f in (0, nf - 1):
        Wf = base[f].reshape(d, q, m)
        for j in (0, q // 2, q - 3, q - 2, q - 1):
            assert rel(Wf[:, j] * (1.0 + f) ** 2, orc.solve_interp(mod, G, grid[j])) <= 1e-10
    for lam in (12, 11, 2):
        solve_lam(lam)
        assert np.array_equal(run(), base), f"forced chunk {lam} differs from the planner's launch"
    solve_lam(0)
    assert np.array_equal(run(), base)


@pytest.fixture
def solve_cluster():
    yield lambda v: call("rp_set_option", b"solve_cluster", v)
    call("rp_set_option", b"solve_cluster", 0)


@pytest.mark.parametrize("m,r,lam", [(10, 2, 2), (10, 2, 12), (1, 2, 8), (16, 3, 8), (3, 2, 0)])
@pytest.mark.parametrize("nf", [1, 3])
def test_eval_solve_clusters_bit_identical(gpu, solve_lam, solve_cluster, m, r, lam, nf):
    """Theta slabs multicast across a cluster of 2/4/8 CTAs (consecutive chunks of one fold, the fold's
    last cluster padded with copies of its last chunk): solutions bit-identical to the unclustered
    solve, every fold and chunk, with W, flags and the (larger, padded) workspace in red zones."""
    d = 200
    q = 41 if m % 2 == 0 else 42
    H, lams_s, tiles1, G, ts, tsh = _solve_setup(d, r, m, seed=40 + m)
    torch = _dev.torch()
    te = tile_elems(d, r + 1)
    tiles = _dev.empty((nf * te,))
    for f in range(nf):  # fold f: the same factors scaled by (1 + f), so every fold's solution differs
        tiles[f * te:(f + 1) * te].copy_(tiles1.reshape(-1)[:te] * (1.0 + f))
    grid = np.logspace(-2, 0, q)
    tv = ts * grid + tsh
    dp = padded(d)
    rhs = _dev.zeros((nf, dp, m))
    rhs[:, :d].copy_(torch.from_numpy(np.ascontiguousarray(G)).unsqueeze(0))
    ldw = q * m + ((q * m) & 1)
    if lam:
        solve_lam(lam)

    def run(cl):
        solve_cluster(cl)
        W = Guarded(nf * dp * ldw)
        fl = Guarded(nf * q)
        ws = guarded_ws(_lib.query("rp_eval_solve_workspace_size", d, r, nf, m, q))
        call("rp_eval_solve", ptr(tiles), d, r, nf, ptr(rhs), m, ptr(_dev.to_dev(tv)), q, ptr(W.buf), ldw,
             ptr(fl.buf), ptr(ws.buf), stream())
        assert W.margins_intact() and fl.margins_intact() and ws.margins_intact(), f"cluster {cl}"
        return W.buf.cpu().numpy().reshape(nf, dp, ldw)[:, :d, :q * m].copy()

    base = run(1)
    mod = orc.fit(H, lams_s, r)
    for f in range(nf):
        Wf = base[f].reshape(d, q, m)
        for j in (0, q // 2, q - 1):  # L scaled by (1+f): W = (LL^T)^-1 G / (1+f)^2
            assert rel(Wf[:, j] * (1.0 + f) ** 2, orc.solve_interp(mod, G, grid[j])) <= 1e-10
    for cl in (2, 4, 8):
        assert np.array_equal(run(cl), base), f"cluster {cl} differs"


def test_generic_solve_matches_specialised_bitwise(gpu):
    """m = 10 with an odd grid size runs the generic kernel for some chunkings; its arithmetic per lambda is
    the specialised kernel's, so results are bit-identical to the fast path on the shared lambdas."""
    d, r, m = 200, 2, 10
    H, lams_s, tiles, G, ts, tsh = _solve_setup(d, r, m, seed=21)
    grid = np.logspace(-2, 0, 24)
    tv = ts * grid + tsh
    fast, _ = _guarded_solve(tiles, d, r, G, tv)
    one = np.stack([_guarded_solve(tiles, d, r, G, tv[j:j + 1])[0][0] for j in range(0, 24, 5)])
    assert np.array_equal(one, fast[0:24:5])


def test_holdout_direct_stays_in_bounds(gpu):
    rng = np.random.default_rng(9)
    nf, n_val, d, m, q = 2, 300, 128, 3, 5
    dp = padded(d)
    X = rng.standard_normal((nf * n_val, d))
    Y = rng.standard_normal((nf * n_val, m))
    ldw = q * m + (q * m & 1)
    Wh = np.zeros((nf, dp, ldw))
    Wh[:, :d, :q * m] = rng.standard_normal((nf, d, q * m))
    dX, dY, dW = _dev.to_dev(X), _dev.to_dev(Y), _dev.to_dev(Wh)
    curves = Guarded(nf * q * m).fill_(0.0)
    ws = guarded_ws(_lib.query("rp_holdout_workspace_size", n_val, d, q, m, nf))
    for metric in (_lib.RP_METRIC_RMSE, _lib.RP_METRIC_MISCLASS):
        call("rp_holdout_direct", ptr(dX), d, n_val, n_val, d, ptr(dY), m, m, ptr(dW), ldw, dp * ldw, q, nf, metric,
             ptr(curves.buf), ptr(ws.buf), stream())
        assert curves.margins_intact() and ws.margins_intact()
        c = curves.buf.cpu().numpy().reshape(nf, q, m)
        for f in range(nf):
            Xv, Yv = X[f * n_val:(f + 1) * n_val], Y[f * n_val:(f + 1) * n_val]
            for j in range(q):
                B = Wh[f, :d, j * m:(j + 1) * m]
                ref = orc.holdout_error(B, Xv, Yv, orc.RMSE if metric == 0 else orc.MISCLASS)
                assert rel(c[f, j], ref) <= 1e-12


@pytest.mark.parametrize("holdout", ["gram", "direct"])
def test_sweeps_are_deterministic(gpu, holdout):
    """Two engines and repeated sweeps on the same data give bit-identical curves (no order-dependent
    atomics, no races between the concurrent Cholesky groups, side streams or tensor-core pipelines)."""
    n, d, m, k, q, s, r = 2560, 256, 4, 5, 21, 4, 2
    X, Y = configs.powerlaw(n, d, m, seed=4)
    grid = orc.make_grid(1e-3, 1e1, q)
    lams, V, _, ts, tsh, P = pichol.fit_basis(grid[orc.sample_indices(q, s)], r)
    dX, dY, tv = _dev.to_dev(X), _dev.to_dev(Y), ts * grid + tsh
    outs = []
    for _ in range(2):
        eng = PicholEngine([n // k] * k, d, m, q, s, r, holdout=holdout)
        for _ in range(2):
            c, _, b = eng.sweep(dX, dY, lams, P, V, tv)
            outs.append((c.cpu().numpy().copy(), b.cpu().numpy().copy()))
    for c, b in outs[1:]:
        assert np.array_equal(c, outs[0][0]) and np.array_equal(b, outs[0][1])


def test_solve_chunk_change_after_allocation(gpu, solve_lam):
    """rp_set_option("solve_lam") after an engine was allocated needs a larger solve workspace for small
    chunks; the engine grows it instead of letting the kernel overrun it, and the curves stay bit-identical."""
    n, d, m, k, q, s, r = 1600, 256, 10, 4, 60, 4, 2
    X, Y = configs.powerlaw(n, d, m, seed=6)
    grid = orc.make_grid(1e-3, 1e1, q)
    lams, V, _, ts, tsh, P = pichol.fit_basis(grid[orc.sample_indices(q, s)], r)
    dX, dY, tv = _dev.to_dev(X), _dev.to_dev(Y), ts * grid + tsh
    eng = PicholEngine([n // k] * k, d, m, q, s, r, holdout="gram")
    base = eng.sweep(dX, dY, lams, P, V, tv)[0].cpu().numpy().copy()
    size0 = eng.ws_solve.numel()
    for lam in (2, 3, 12):
        solve_lam(lam)
        c = eng.sweep(dX, dY, lams, P, V, tv)[0].cpu().numpy()
        assert np.array_equal(c, base), lam
    assert eng.ws_solve.numel() >= size0
