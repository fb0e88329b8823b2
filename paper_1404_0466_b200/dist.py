"""Fold sharding across the GPUs of one node.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch). Folds are
independent until the final mean. When k % world == 0 rank r owns the contiguous
folds r*k/world .. (r+1)*k/world - 1, which are also the row blocks whose Gram it
computes, so it uploads only those rows of X (1/world of the design); otherwise
fold f runs on rank f % world with every block replicated. Two exchanges are
real data dependencies of the path:

* Gram blocks: the training Hessian of fold f is sum_{b != f} G_b, so every
  rank needs all k fold-block Grams. When k % world == 0 each rank computes only
  its own k / world blocks and the blocks are all-gathered (deterministic: every
  rank then sums them in the same fixed order, so H_f is bit-identical at any
  GPU count). Otherwise every rank computes all blocks (replicated, no exchange).
* Curves: the (q x m) per-fold error curves are all-gathered (16 KB per fold at
  c4) and every rank runs the same ordered fold mean + argmin.

The hooks operate on torch tensors only, so the same code runs on CPU tensors
with the gloo backend (tests/test_dist_gloo.py), and on CUDA tensors over gloo
by staging through host memory (two ranks sharing one GPU in
tests/test_gpu_dist.py; NCCL is the backend on a multi-GPU node).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass
class Shard:
    rank: int
    world: int
    k: int

    @property
    def exchange(self):
        return self.world > 1 and self.k % self.world == 0

    def owner(self, f):
        """Rank that computes fold f: the owner of block f when blocks are exchanged (contiguous
        runs of k / world folds, so a rank's folds are its own Gram blocks and it needs no other
        rows of X), round-robin otherwise."""
        return f // (self.k // self.world) if self.exchange else f % self.world

    def slot(self, f):
        """Position of fold f among its owner's local folds."""
        return f % (self.k // self.world) if self.exchange else f // self.world

    @property
    def local_folds(self):
        return [f for f in range(self.k) if self.owner(f) == self.rank]

    @property
    def gram_blocks(self):
        """Blocks whose Gram this rank computes (none for a rank without folds when the blocks
        are replicated: world > k leaves ranks k..world-1 with only the curve exchange)."""
        if not self.exchange:
            return list(range(self.k)) if self.local_folds else []
        per = self.k // self.world
        return list(range(self.rank * per, (self.rank + 1) * per))

    @property
    def needed_blocks(self):
        """Row blocks of X / Y this rank reads: its Gram blocks and its folds' validation rows."""
        return sorted(set(self.gram_blocks) | set(self.local_folds))

    @property
    def slots(self):
        """Curves gathered per rank (ranks with fewer folds pad to this)."""
        return -(-self.k // self.world)


def _host_staged(t, group=None):
    """True when the process group cannot run collectives on ``t``'s device (gloo with CUDA
    tensors: the exchange is staged through pinned host memory instead)."""
    import torch.distributed as dist

    return t.is_cuda and dist.get_backend(group) == "gloo"


def _all_gather_into(out, mine, group=None):
    import torch.distributed as dist

    if _host_staged(out, group):
        host = out.new_empty(out.shape, device="cpu")
        dist.all_gather_into_tensor(host, mine.cpu(), group=group)
        out.copy_(host)
    else:
        dist.all_gather_into_tensor(out, mine, group=group)


def exchange_grams(shard, G, C, yy=None, group=None):
    """All-gather contiguous Gram blocks so every rank holds all k (G: (k, d, d), C: (k, m, d))."""
    if not shard.exchange:
        return
    per = shard.k // shard.world
    lo = shard.rank * per
    for buf in (G, C) + ((yy,) if yy is not None else ()):
        mine = buf[lo : lo + per].clone()
        _all_gather_into(buf, mine, group=group)


def gather_curves(shard, curves_local, group=None):
    """All-gather per-fold curves (nf_local, q, m) into fold order (k, q, m)."""
    import torch

    if shard.world == 1:
        return curves_local
    nf, q, m = curves_local.shape
    slots = shard.slots
    pad = torch.zeros((slots, q, m), dtype=curves_local.dtype, device=curves_local.device)
    pad[:nf].copy_(curves_local)
    out = torch.empty((shard.world * slots, q, m), dtype=curves_local.dtype, device=curves_local.device)
    _all_gather_into(out, pad, group=group)
    order = [shard.owner(f) * slots + shard.slot(f) for f in range(shard.k)]
    return out[torch.as_tensor(order, device=out.device)].contiguous()


def ordered_select(curves_all):
    """Fold mean in fold order then first argmin per output (cvsearch.py:154-175), on any device."""
    import torch

    k = curves_all.shape[0]
    s = curves_all[0].clone()
    for f in range(1, k):
        s += curves_all[f]
    mean = s / k
    best = torch.argmin(mean, dim=0)
    return mean, best
