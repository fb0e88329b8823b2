"""CPU baseline modes of SURVEY.md 8(d) / BASELINE.md 4 on the box's host cores (run once per round on the
GPU box; the result is committed under profiles/ and quoted by bench.py's cpu_baseline["modes"]).

    python tools/cpu_modes.py [config] > profiles/rNN_cpu_modes.json

The oracle port (oracle/pichol_oracle.py, the reference package restated; the reference itself is pure
Python and does not travel to the box) is timed on a bounded sample of the config's workload, in three modes:

* ``multi_rhs_all_threads``: the multi-RHS composition (one fit per fold, every output solved per lambda),
  BLAS on all host threads -- the mode bench.py's live cpu_baseline uses;
* ``stock_per_output``: the reference driver as shipped (cvsearch.py:206-243 is single-target), run once per
  output: per fold assemble + fit + q x (solve_interp + holdout_error) with one right-hand side, all BLAS
  threads; the m-output sweep costs m such runs;
* ``fold_threads_blas1``: the reference's own parallel mode (``threads=k``, cvsearch.py:126-142 /
  cli.py:322): k folds on a thread pool, BLAS limited to one thread per call (threadpoolctl).

Each mode times the per-fold setup and a few lambdas, then extrapolates linearly to the whole sweep (k folds
x q lambdas); value = fold-lambda evals/s where one eval covers all m outputs (bench.py's metric).
"""

import json
import os
import platform
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from oracle import pichol_oracle as orc  # noqa: E402
from paper_1404_0466_b200 import configs  # noqa: E402


def host_info():
    model = platform.processor()
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = []
    try:
        from threadpoolctl import threadpool_info

        blas = [{k: v for k, v in i.items() if k in ("internal_api", "version", "num_threads", "threading_layer")}
                for i in threadpool_info()]
    except ImportError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            "numpy": np.__version__, "blas": blas}


def fold_sample(cfg, X, Y, fold, n_lam, single=False):
    grid = orc.make_grid(cfg.lo, cfg.hi, cfg.q)
    assign = np.arange(cfg.n) // (cfg.n // cfg.k)
    val = assign == fold
    Yc = Y[:, :1] if single else Y
    t0 = time.perf_counter()
    H, G = orc.assemble(X[~val], Yc[~val])
    model = orc.fit(H, grid[orc.sample_indices(cfg.q, cfg.s)], cfg.r)
    t1 = time.perf_counter()
    for li in np.linspace(0, cfg.q - 1, n_lam).round().astype(int):
        B = orc.solve_interp(model, G, grid[li])
        orc.holdout_error(B, X[val], Yc[val])
    t2 = time.perf_counter()
    return t1 - t0, (t2 - t1) / n_lam


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    n_lam = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cfg = configs.CONFIGS[name]
    X, Y = configs.generate(cfg)
    k, q, m = cfg.k, cfg.q, cfg.m
    out = {"config": name, "host": host_info(), "modes": {}}
    warm = configs.CONFIGS["c1"]  # page in BLAS / scipy before the first timed sample
    fold_sample(warm, *configs.generate(warm), 0, 1)

    ts, tl = fold_sample(cfg, X, Y, 0, n_lam)
    out["modes"]["multi_rhs_all_threads"] = {
        "value": q / (ts + q * tl), "t_setup_s": ts, "t_lambda_s": tl, "cores": os.cpu_count(),
        "sample": f"fold 0: assemble + {cfg.s} Choleskys + fit + {n_lam} lambdas (m={m} RHS), extrapolated"}

    ts1, tl1 = fold_sample(cfg, X, Y, 0, n_lam, single=True)
    out["modes"]["stock_per_output"] = {
        "value": q / (m * (ts1 + q * tl1)), "t_setup_s": ts1, "t_lambda_s": tl1, "cores": os.cpu_count(),
        "sample": f"fold 0, output 0: the stock single-target driver's fold work + {n_lam} lambdas, extrapolated "
                  f"to k={k} folds x q={q} lambdas x m={m} outputs (one driver run per output)"}

    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        with ThreadPoolExecutor(max_workers=k) as pool:
            res = list(pool.map(lambda f: fold_sample(cfg, X, Y, f, n_lam), range(k)))
        wall = time.perf_counter() - t0
    setup = max(r[0] for r in res)
    lam = max(r[1] for r in res)
    # the folds run concurrently (in waves when k exceeds the cores): the sweep's wall time ~ waves x the
    # slowest fold's setup + q lambdas
    waves = -(-k // (os.cpu_count() or 1))
    out["modes"]["fold_threads_blas1"] = {
        "value": k * q / (waves * (setup + q * lam)), "t_setup_s_max": setup, "t_lambda_s_max": lam, "sample_wall_s": wall,
        "cores": min(k, os.cpu_count()),
        "sample": f"k={k} folds concurrently on a thread pool, 1 BLAS thread each: setup + {n_lam} lambdas per "
                  f"fold, extrapolated to q={q} lambdas"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
