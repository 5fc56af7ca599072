"""Multi-GPU query serving: replicas with query-column sharding.

Katz queries are independent columns, so N GPUs each hold a
full replica of the index and solve a contiguous slice of the query batch;
there is no exchange inside a solve.  The only collective is the final
gather of the (small) ranked results, done with torch.distributed
(NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np


def shard(items, world, rank):
    """Contiguous, order-preserving slice of `items` for `rank`."""
    items = np.asarray(items)
    bounds = np.linspace(0, items.size, world + 1).astype(np.int64)
    return items[bounds[rank] : bounds[rank + 1]]


def gather_in_order(local, world, group=None):
    """all_gather_object of per-rank result lists, concatenated in rank order."""
    import torch.distributed as dist

    if world == 1:
        return list(local)
    parts = [None] * world
    dist.all_gather_object(parts, list(local), group=group)
    out = []
    for p in parts:
        out.extend(p)
    return out


def sharded(fn, qs, *args, group=None, **kw):
    """Run fn(shard_of_qs, *args, **kw) -> list on every rank and return the
    full list (query order) on every rank."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    else:
        world, rank = 1, 0
    mine = shard(qs, world, rank)
    local = fn(mine, *args, **kw) if mine.size else []
    return gather_in_order(local, world, group)


def katz_rank_distributed(idx, qs, s, tol=1e-10, group=None):
    """katz_rank_batch over all ranks' GPUs (each rank holds `idx`)."""
    from .linkpred import katz_rank_batch

    return sharded(lambda q: katz_rank_batch(idx, q, s, tol), qs, group=group)


def sparse_katz_distributed(idx, qs, s, T=None, tol=1e-10, group=None):
    """sparse_katz_batch over all ranks' GPUs."""
    from .linkpred import sparse_katz_batch

    return sharded(lambda q: sparse_katz_batch(idx, q, s, T, tol), qs, group=group)
