"""Golden fixtures for the command line and the matrix files, made by running the REAL
reference CLI (ridgepath.cli.main) in the build container:

    python tests/golden/make_cli_golden.py

Writes tests/golden/cli/: input matrices saved by the reference's matio (RPMATX01 + CSV),
and the reference's CSV reports and stdout lines for `cv --method pichol|chol` and
`factor-path`. Timing columns and wall seconds vary run to run; the tests compare the rest.
"""

import contextlib
import io
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cli")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from ridgepath import cli, matio  # noqa: E402

from paper_1404_0466_b200 import configs  # noqa: E402


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, buf.getvalue().strip()


def main():
    os.makedirs(OUT, exist_ok=True)
    X, Y = configs.powerlaw(300, 20, 1, seed=11)
    Xm, Ym = configs.maclaurin(240, 16, m=1, seed=5)
    H = X.T @ X / 300.0
    p = lambda name: os.path.join(OUT, name)  # noqa: E731
    matio.save_matrix(p("X.bin"), X)
    matio.save_matrix(p("y.bin"), Y)
    matio.save_csv(p("X.csv"), X)
    matio.save_csv(p("y.csv"), Y)
    matio.save_matrix(p("Xm.bin"), Xm)
    matio.save_matrix(p("ym.bin"), Ym)
    matio.save_matrix(p("H.bin"), H)
    runs = {
        "cv_pichol": ["cv", "--x", p("X.bin"), "--y", p("y.bin"), "--method", "pichol", "--lo", "1e-3", "--hi", "10",
                      "--q", "15", "--folds", "4", "--fold-seed", "3"],
        "cv_chol": ["cv", "--x", p("X.csv"), "--y", p("y.csv"), "--method", "chol", "--lo", "1e-3", "--hi", "10",
                    "--q", "15", "--folds", "4", "--fold-seed", "3"],
        "cv_mis": ["cv", "--x", p("Xm.bin"), "--y", p("ym.bin"), "--method", "pichol", "--metric", "misclass",
                   "--q", "11", "--folds", "3", "--g", "3", "--r", "2"],
        "cv_mchol": ["cv", "--x", p("X.bin"), "--y", p("y.bin"), "--method", "mchol", "--lo", "1e-3", "--hi", "10",
                     "--q", "15", "--folds", "4", "--fold-seed", "3"],
        "cv_pinrmse": ["cv", "--x", p("X.bin"), "--y", p("y.bin"), "--method", "pinrmse", "--lo", "1e-3", "--hi",
                       "10", "--q", "15", "--folds", "4", "--fold-seed", "3", "--g", "5", "--r", "2"],
        "fp": ["factor-path", "--matrix", p("H.bin"), "--lambdas", "0.01,0.03,0.1,0.3,1,3", "--g", "4", "--r", "2"],
    }
    stdout = {}
    for name, argv in runs.items():
        rc, line = run(argv + ["--out", p(name + ".csv"), "--no-figures"])
        assert rc == 0, (name, rc)
        stdout[name] = {"argv": [a.replace(OUT + "/", "") for a in argv], "rc": rc, "stdout": line}
    # error exits
    stdout["bad_shape"] = {"rc": cli.main(["cv", "--x", p("X.bin"), "--y", p("H.bin"), "--method", "pichol",
                                           "--no-figures", "--out", "/tmp/x.csv"])}
    stdout["missing_file"] = {"rc": cli.main(["cv", "--x", p("nope.bin"), "--y", p("y.bin"), "--method", "pichol",
                                              "--no-figures", "--out", "/tmp/x.csv"])}
    stdout["bad_arg"] = {"rc": cli.main(["cv", "--x", p("X.bin")])}
    with open(p("runs.json"), "w") as f:
        json.dump(stdout, f, indent=1)
    print(json.dumps(stdout, indent=1))


if __name__ == "__main__":
    main()
