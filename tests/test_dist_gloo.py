"""Multi-process (world_size 2, gloo, CPU) test of the fold-sharding host logic in
paper_1404_0466_b200/dist.py: fold placement, the Gram-block all-gather, the curve
all-gather into fold order and the ordered selection. The per-fold arithmetic is the
CPU oracle standing in for the device (this test exercises the exchange, not kernels);
the merged result must equal the single-process result bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pichol_oracle as orc
from paper_1404_0466_b200 import configs
from paper_1404_0466_b200.dist import Shard, exchange_grams, gather_curves, ordered_select

N, D, M, K, Q, S, R = 480, 12, 3, 4, 9, 4, 2


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fold_curves(X, Y, Gblocks, Cblocks, f, grid):
    """Per-fold curve from Gram blocks (sum_{b != f} G_b in block order), like the device pipeline."""
    H = sum(Gblocks[b] for b in range(K) if b != f)
    G = sum(Cblocks[b] for b in range(K) if b != f)
    model = orc.fit(H, grid[orc.sample_indices(Q, S)], R)
    rows = slice(f * (N // K), (f + 1) * (N // K))
    return np.stack([orc.holdout_error(orc.solve_interp(model, G, lam), X[rows], Y[rows]) for lam in grid])


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, Y = configs.powerlaw(N, D, M, seed=5)
    grid = orc.make_grid(1e-3, 1e1, Q)
    shard = Shard(rank, world, K)
    G = torch.zeros((K, D, D), dtype=torch.float64)
    C = torch.zeros((K, M, D), dtype=torch.float64)
    for b in shard.gram_blocks:  # this rank's blocks only
        rows = slice(b * (N // K), (b + 1) * (N // K))
        G[b] = torch.from_numpy(X[rows].T @ X[rows])
        C[b] = torch.from_numpy((X[rows].T @ Y[rows]).T)
    exchange_grams(shard, G, C)
    Gb = [G[b].numpy() for b in range(K)]
    Cb = [C[b].numpy().T for b in range(K)]
    local = torch.from_numpy(np.stack([_fold_curves(X, Y, Gb, Cb, f, grid) for f in shard.local_folds]))
    curves = gather_curves(shard, local)
    mean, best = ordered_select(curves)
    if rank == 0:
        out["curves"] = curves.numpy().copy()
        out["mean"] = mean.numpy().copy()
        out["best"] = best.numpy().copy()
        out["G"] = G.numpy().copy()
    dist.barrier()
    dist.destroy_process_group()


def _single():
    X, Y = configs.powerlaw(N, D, M, seed=5)
    grid = orc.make_grid(1e-3, 1e1, Q)
    Gb, Cb = [], []
    for b in range(K):
        rows = slice(b * (N // K), (b + 1) * (N // K))
        Gb.append(X[rows].T @ X[rows])
        Cb.append(X[rows].T @ Y[rows])
    curves = np.stack([_fold_curves(X, Y, Gb, Cb, f, grid) for f in range(K)])
    mean, best = ordered_select(torch.from_numpy(curves))
    return curves, mean.numpy(), best.numpy(), np.stack(Gb)


def test_shard_placement():
    for world in (1, 2, 4, 8):
        seen = sorted(f for r in range(world) for f in Shard(r, world, 8).local_folds)
        assert seen == list(range(8))
    s = Shard(1, 4, 5)
    assert s.local_folds == [1] and not s.exchange and s.gram_blocks == list(range(5))
    s = Shard(1, 2, 8)
    assert s.local_folds == [4, 5, 6, 7] and s.exchange and s.gram_blocks == [4, 5, 6, 7]
    assert s.needed_blocks == [4, 5, 6, 7] and Shard(3, 8, 8).needed_blocks == [3]
    assert Shard(1, 3, 5).needed_blocks == list(range(5))
    # world > k (c1-c3 have k = 5 on an 8-GPU node): ranks without folds compute nothing and only
    # join the curve exchange
    s = Shard(6, 8, 5)
    assert s.local_folds == [] and not s.exchange and s.gram_blocks == [] and s.slots == 1


def test_two_rank_gloo_matches_single_process():
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(2, _port(), out), nprocs=2, join=True)
        res = dict(out)
    curves, mean, best, G = _single()
    assert np.array_equal(res["G"], G)  # exchanged blocks are exact copies
    assert np.array_equal(res["curves"], curves)  # bit-identical at any world size
    assert np.array_equal(res["mean"], mean)
    assert np.array_equal(res["best"], best)
    # and the oracle's own merge gives the same selection
    assert np.array_equal(orc.merge(curves)[1], best)
