"""CPU-only checks: the C-ABI library loads and exports every declared symbol, argument
validation fails with the reference's exception types, and the host-side logic of the
drop-in (layouts, basis, folds, report) matches the reference / oracle. No compute call
touches a GPU here."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import pichol_oracle as orc
from paper_1404_0466_b200 import _lib, configs, cvsearch, errors, pichol, trivec
from tests.conftest import golden

HEADER = os.path.join(os.path.dirname(__file__), "..", "include", "ridgepath_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_queries_without_gpu():
    assert _lib.query("rp_version") == 1
    assert _lib.query("rp_tile_count", 4096) == 64 * 65 // 2
    assert _lib.query("rp_tile_count", 65) == 3
    assert _lib.query("rp_potrf_workspace_size", 4096, 40) == 40 * 128 * 128 * 8
    assert _lib.query("rp_launch_count") >= 0


def test_invalid_arguments_map_to_usage_errors():
    # validation happens before any CUDA call, so this runs on the CPU box
    with pytest.raises(errors.DimensionMismatch):
        _lib.call("rp_eval_solve", None, 0, 2, 1, None, 1, None, 1, None, 2, None, None, None)
    with pytest.raises(errors.UsageError):
        _lib.call("rp_eval_solve", None, 64, 9, 1, None, 1, None, 1, None, 2, None, None, None)
    with pytest.raises(errors.UsageError):
        _lib.call("rp_potrf_batched", None, 0, 0, 1, None, None, None)
    assert "rp_potrf_batched" in _lib.last_error()


def test_compute_entry_points_fail_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(errors.DeviceError):
        from paper_1404_0466_b200 import linalg

        linalg.cholesky(np.eye(3))


# ---------------------------------------------------------------- layouts (trivec.py)


def pack_positions(layout):
    return [(int(i) % layout.h, int(i) // layout.h) for i in layout.perm]


def test_frozen_orders_of_the_reference_tests():
    # restated from the reference's tests/test_trivec.py:23-62
    assert pack_positions(trivec.build_layout(trivec.ROWWISE, 3)) == [(0, 0), (1, 0), (1, 1), (2, 0), (2, 1), (2, 2)]
    assert pack_positions(trivec.build_layout(trivec.RECURSIVE, 4, h0=2)) == [
        (2, 0), (3, 0), (2, 1), (3, 1), (0, 0), (1, 0), (1, 1), (2, 2), (3, 2), (3, 3)]
    assert pack_positions(trivec.build_layout(trivec.RECURSIVE, 5, h0=4))[:6] == [
        (3, 0), (4, 0), (3, 1), (4, 1), (3, 2), (4, 2)]


def test_layout_perms_match_reference_golden():
    g = golden("layouts")
    for key in g.files:
        parts = key.split("_")
        if parts[0] == "recursive":
            lay = trivec.build_layout(trivec.RECURSIVE, int(parts[1]), int(parts[2]))
        else:
            lay = trivec.build_layout(trivec.ROWWISE, int(parts[1]))
        assert np.array_equal(lay.perm, g[key]), key


def test_layout_bijection_and_index_of():
    for kind in (trivec.ROWWISE, trivec.RECURSIVE, trivec.TILE):
        for h in (1, 2, 7, 63, 64, 65, 130):
            lay = trivec.build_layout(kind, h)
            assert lay.length == h * (h + 1) // 2
            r, c = np.tril_indices(h)
            assert np.array_equal(np.sort(lay.perm), np.sort(c * h + r)), (kind, h)
    lay = trivec.build_layout(trivec.RECURSIVE, 9, h0=4)
    assert lay.index_of(8, 0) == int(np.flatnonzero(lay.perm == 0 * 9 + 8)[0])
    with pytest.raises(errors.UsageError):
        lay.index_of(0, 1)


@pytest.mark.parametrize("kind,h,h0", [("rowwise", 1, 64), ("rowwise", 100, 64), ("recursive", 257, 16),
                                       ("recursive", 64, 64), ("tile", 130, 64)])
def test_copy_plan_reassembles_the_permutation(kind, h, h0):
    """copy_plan (trivec.py:100-120): slice runs of at least the threshold length plus element gathers
    that together rebuild perm exactly, each destination covered once."""
    lay = trivec.build_layout(kind, h, h0)
    run_src, run_dst, run_len, gat_dst, gat_src = lay.copy_plan()
    out = np.full(lay.length, -1, dtype=np.int64)
    hits = np.zeros(lay.length, dtype=np.int64)
    for s0, d0, n0 in zip(run_src, run_dst, run_len):
        out[d0:d0 + n0] = np.arange(s0, s0 + n0)
        hits[d0:d0 + n0] += 1
    out[gat_dst] = gat_src
    hits[gat_dst] += 1
    assert np.array_equal(out, lay.perm) and np.all(hits == 1)
    assert np.all(run_len >= trivec._RUN_THRESHOLD)


def test_layout_validation():
    with pytest.raises(errors.UsageError):
        trivec.build_layout("diagonal", 4)
    with pytest.raises(errors.UsageError):
        trivec.build_layout(trivec.ROWWISE, 0)
    with pytest.raises(errors.UsageError):
        trivec.build_layout(trivec.RECURSIVE, 4, h0=0)


# ---------------------------------------------------------------- host half of the fit


@pytest.mark.parametrize("lams,r", [([0.05, 0.2, 0.7, 2.0], 2), (1e4 + np.linspace(0, 1e-3, 5), 2),
                                    (np.logspace(-5, 3, 6), 3), ([1.0, 4.0, 9.0], 1)])
def test_fit_basis_matches_oracle(lams, r):
    ls, V, cond, ts, tsh, P = pichol.fit_basis(lams, r)
    ols, oV, ocond, ots, otsh = orc.fit_basis(lams, r)
    assert np.array_equal(ls, ols) and np.array_equal(V, oV)
    assert cond == ocond and ts == ots and tsh == otsh
    # P = (V^T V)^{-1} V^T: P V = I
    assert np.max(np.abs(P @ V - np.eye(r + 1))) <= 1e-6 * np.linalg.cond(V) ** 2 * 1e-10 + 1e-9


def test_fit_basis_scalar_closed_form():
    # reference tests/test_pichol.py:21-27: samples {1,4,9}, sqrt targets -> theta = (6/7, 12/49)
    ls, V, cond, ts, tsh, P = pichol.fit_basis([1.0, 4.0, 9.0], 1)
    theta = P @ np.array([1.0, 2.0, 3.0])
    assert np.allclose(theta, [6.0 / 7.0, 12.0 / 49.0], atol=1e-12)
    assert ts == 1.0 and tsh == 0.0


def test_sample_indices_and_grid_match_reference_semantics():
    assert np.array_equal(pichol.sample_indices(31, 4), [0, 10, 20, 30])
    assert np.array_equal(pichol.sample_indices(4, 4), [0, 1, 2, 3])
    g = cvsearch.make_grid(1e-3, 1.0, 31)
    assert g.values[0] == 1e-3 and g.values[-1] == 1.0
    assert cvsearch.make_grid(0.5, 1.0, 1).values.tolist() == [0.5]
    for bad in ((1.0, 0.5, 5), (0.0, 1.0, 5), (0.1, 1.0, 0)):
        with pytest.raises(errors.UsageError):
            cvsearch.make_grid(*bad)


def test_make_folds_matches_reference_semantics():
    f1 = cvsearch.make_folds(103, 5, seed=7)
    assert np.array_equal(f1.assignments, cvsearch.make_folds(103, 5, seed=7).assignments)
    sizes = np.bincount(f1.assignments, minlength=5)
    assert sizes.max() - sizes.min() <= 1
    labels = np.array([1.0] * 12 + [-1.0] * 8)
    folds = cvsearch.make_folds(20, 4, seed=0, labels=labels)
    for k in range(4):
        val = folds.assignments == k
        assert np.sum(labels[val] == 1.0) == 3 and np.sum(labels[val] == -1.0) == 2
    with pytest.raises(errors.UsageError):
        cvsearch.make_folds(10, 1, seed=0)


def test_fold_order_is_stable_grouping():
    folds = cvsearch.make_folds(50, 4, seed=3)
    order, counts = cvsearch.fold_order(folds, 50)
    assert order is not None
    a = folds.assignments[order]
    assert np.all(np.diff(a) >= 0)
    for f in range(4):
        rows = order[a == f]
        assert np.all(np.diff(rows) > 0)  # original row order kept inside a fold
    assert counts.tolist() == np.bincount(folds.assignments).tolist()
    order, counts = cvsearch.fold_order(cvsearch.contiguous_folds(40, 4), 40)
    assert order is None and counts.tolist() == [10] * 4


def test_merge_and_csv_schema():
    rng = np.random.default_rng(0)
    grid = cvsearch.make_grid(0.01, 0.1, 5)
    curves = rng.random((3, 5, 1))
    curves[:, 2, 0] = 0.0  # ties -> first minimum
    curves[:, 3, 0] = 0.0
    times = dict.fromkeys(cvsearch.PHASES, 0.5)
    rep = cvsearch._merge("pichol", grid.values, curves, times, 1.0)
    assert rep.best_lambda == grid.values[2]
    assert rep.best_error == 0.0
    lines = cvsearch.report_csv_lines(rep)
    assert lines[0] == "method,fold,lambda,error,t_factorize,t_vec,t_fit,t_interp,t_solve,t_predict"
    assert len(lines) == 1 + 3 * 5 + 5
    mean_rows = [l for l in lines[1:] if l.split(",")[1] == "-1"]
    for row in mean_rows:
        cells = row.split(",")
        assert float(cells[3]) == rep.per_lambda_error[float(cells[2])]
        assert all(float(c) == 0.0 for c in cells[4:])
    assert np.array_equal(rep.per_lambda_error[float(grid.values[0])], np.mean(curves[:, 0, 0]))


def test_resolve_threads(monkeypatch):
    monkeypatch.delenv(cvsearch.THREADS_ENV, raising=False)
    assert cvsearch.resolve_threads(None) == 1
    monkeypatch.setenv(cvsearch.THREADS_ENV, "zebra")
    with pytest.raises(errors.UsageError):
        cvsearch.resolve_threads(None)


def test_configs_match_baseline_shapes():
    c = configs.CONFIGS
    assert (c["c4"].n, c["c4"].d, c["c4"].m, c["c4"].k, c["c4"].s, c["c4"].r, c["c4"].q) == (100000, 4096, 10, 8, 5,
                                                                                                  2, 200)
    assert (c["c5"].d, c["c5"].m, c["c5"].s, c["c5"].r, c["c5"].q, c["c5"].lo, c["c5"].hi) == (8192, 16, 6, 3, 500, 1e-5,
                                                                                                  1e3)
    X, Y = configs.maclaurin(300, 64, m=10, seed=0)
    assert X.shape == (300, 64) and set(np.unique(Y)) == {-1.0, 1.0}
    assert np.all(np.sum(Y == 1.0, axis=1) == 1)


def test_error_taxonomy_matches_reference():
    assert errors.UsageError.exit_code == 1 and errors.NumericalError.exit_code == 2 and errors.IoError.exit_code == 3
    assert issubclass(errors.DimensionMismatch, errors.UsageError)
    assert issubclass(errors.SingularInterpolant, errors.NumericalError)
    assert issubclass(errors.NotPositiveDefinite, errors.NumericalError)
    assert issubclass(errors.EmptyValidationSet, errors.UsageError)
