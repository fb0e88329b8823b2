"""The fold-sharded sweep for real: several ranks (processes) drive the device path on the one GPU
this pool provides, exchanging Gram blocks and curves over torch.distributed (gloo, staged through
host memory -- NCCL on a multi-GPU node). Each rank runs only its folds and, when k % world == 0,
only its Gram blocks (its folds are then those same blocks, and it uploads only their rows); the merged curves and selection must be bit-identical
to the single-process sweep (fixed per-fold arithmetic, fixed-order sums; the reference's own
contract, cvsearch.py:137-142 and tests/test_cvsearch.py:168-178). world > k leaves ranks without
folds that only join the curve exchange.

The ranks do not wait on each other inside kernels (each exchange is a host-side collective), so
sharing one GPU is a functional test of the sharded path, not a stand-in for multi-GPU timing."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1404_0466_b200 import configs

pytestmark = pytest.mark.gpu

N, D, M, Q, S, R = 2400, 256, 3, 13, 4, 2


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(k):
    cfg = configs.CONFIGS["c4"].scaled(n=N, d=D, m=M, q=Q, s=S, r=R, k=k)
    X, Y = configs.generate(cfg)
    return cfg, X, Y, configs.grid_values(cfg)


def _worker(rank, world, k, port, out):
    import torch.distributed as dist

    from paper_1404_0466_b200 import cvsearch
    from paper_1404_0466_b200.dist import Shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, X, Y, grid = _inputs(k)
    shard = Shard(rank, world, k)
    sess = cvsearch.CvSession([cfg.n // k] * k, cfg.d, cfg.m, grid, g=cfg.s, r=cfg.r, shard=shard)
    curves, best = sess.run(X, Y)  # pageable numpy: blocking per-block copies of the needed rows
    # pinned host tensors: the streamed per-block upload of only this rank's rows
    c2, b2 = sess.run(torch.from_numpy(X).pin_memory(), torch.from_numpy(Y).pin_memory())
    assert np.array_equal(c2, curves) and np.array_equal(b2, best)
    rows = sum(cfg.n // k for _ in shard.needed_blocks)
    assert sess.h2d_bytes == rows * (cfg.d + cfg.m) * 8
    out[rank] = (curves.copy(), best.copy(), list(shard.local_folds), list(sess.engine.gram_blocks),
                 list(shard.needed_blocks))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k", [(2, 4), (2, 3), (3, 2)])
def test_sharded_ranks_match_single_process(gpu, world, k):
    from paper_1404_0466_b200 import cvsearch

    cfg, X, Y, grid = _inputs(k)
    ref_curves, ref_best = cvsearch.CvSession([cfg.n // k] * k, cfg.d, cfg.m, grid, g=cfg.s, r=cfg.r).run(X, Y)
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, k, _port(), out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        curves, best, folds, blocks, needed = res[rank]
        if k % world == 0:  # contiguous folds = the rank's own Gram blocks
            assert folds == list(range(rank * (k // world), (rank + 1) * (k // world)))
        else:
            assert folds == [f for f in range(k) if f % world == rank]
        if k % world == 0:
            assert len(blocks) == k // world  # Gram blocks computed locally, the rest exchanged
            assert needed == blocks  # and only those rows of X / Y uploaded
        assert np.array_equal(curves, ref_curves), rank
        assert np.array_equal(best, ref_best), rank
