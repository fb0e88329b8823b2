"""Matrix files and the command line on the host (no GPU): RPMATX01/CSV against files the
reference's matio wrote (tests/golden/make_cli_golden.py), and the CLI's argument handling
and exit codes (cli.py:315-329) up to the first device call."""

import json
import os

import numpy as np
import pytest

from paper_1404_0466_b200 import cli, matio
from paper_1404_0466_b200.errors import BadFormat, IoError

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cli")


def gp(name):
    return os.path.join(GOLD, name)


def test_reference_files_load_and_agree():
    X = matio.load_matrix(gp("X.bin"))
    assert X.shape == (300, 20) and X.flags.f_contiguous
    assert np.array_equal(X, matio.load_csv(gp("X.csv")))  # %.17g text round-trips exactly
    assert np.array_equal(matio.load_any(gp("y.bin")), matio.load_any(gp("y.csv")))


def test_save_matrix_is_byte_identical(tmp_path):
    X = matio.load_matrix(gp("X.bin"))
    out = tmp_path / "X.bin"
    matio.save_matrix(str(out), X)
    assert out.read_bytes() == open(gp("X.bin"), "rb").read()
    matio.save_matrix(str(out), np.ascontiguousarray(X))  # C-ordered input, same bytes
    assert out.read_bytes() == open(gp("X.bin"), "rb").read()


def test_csv_round_trip(tmp_path):
    a = np.random.default_rng(0).standard_normal((7, 3))
    matio.save_csv(str(tmp_path / "a.csv"), a)
    assert np.array_equal(matio.load_any(str(tmp_path / "a.csv")), a)


def test_load_design_pinned_row_major_and_permuted():
    X = matio.load_matrix(gp("X.bin"))
    Xp, shape = matio.load_design_pinned(gp("X.bin"))
    assert shape == X.shape and Xp.is_contiguous()
    assert np.array_equal(Xp.numpy(), X)
    order = np.random.default_rng(1).permutation(X.shape[0])
    Xo, _ = matio.load_design_pinned(gp("X.bin"), order=order)
    assert np.array_equal(Xo.numpy(), X[order])


def test_bad_files(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTMAGIC" + bytes(16))
    with pytest.raises(BadFormat):
        matio.load_matrix(str(bad))
    trunc = tmp_path / "trunc.bin"
    trunc.write_bytes(open(gp("H.bin"), "rb").read()[:-8])
    with pytest.raises(BadFormat):
        matio.load_matrix(str(trunc))
    with pytest.raises(BadFormat):
        matio.load_design_pinned(str(trunc))
    with pytest.raises(IoError):
        matio.load_matrix(str(tmp_path / "missing.bin"))
    with pytest.raises(BadFormat):
        matio.save_matrix(str(tmp_path / "v.bin"), np.zeros(3))


def test_exit_codes_match_reference(tmp_path):
    runs = json.load(open(gp("runs.json")))
    out = str(tmp_path / "r.csv")
    rc = cli.main(["cv", "--x", gp("X.bin"), "--y", gp("H.bin"), "--method", "pichol", "--no-figures", "--out", out])
    assert rc == runs["bad_shape"]["rc"] == 1
    rc = cli.main(["cv", "--x", gp("nope.bin"), "--y", gp("y.bin"), "--method", "pichol", "--no-figures", "--out", out])
    assert rc == runs["missing_file"]["rc"] == 3
    assert cli.main(["cv", "--x", gp("X.bin")]) == runs["bad_arg"]["rc"] == 1
    # baselines outside the hot path and other reference commands: usage errors
    assert cli.main(["cv", "--x", gp("X.bin"), "--y", gp("y.bin"), "--method", "svd", "--out", out]) == 1
    assert cli.main(["cv", "--x", gp("X.bin"), "--y", gp("y.bin"), "--method", "rsvd", "--out", out]) == 1
    assert cli.main(["gen", "--n", "10"]) == 1
    assert cli.main(["--help"]) == 0
