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


def sparse_katz_distributed(idx, qs, s, T=None, tol=1e-10, group=None, engine=None):
    """sparse_katz over all ranks' GPUs with the anchor solves deduplicated
    across the whole batch.

    1. every rank solves its contiguous shard of the queries and selects their
       candidates and anchors (stage 1 of linkpred.SparseKatzEngine);
    2. the small per-query tables (anchor ids, candidate ids, counts) are
       all-gathered; the globally unique anchor list is cut into contiguous
       shares, one per rank;
    3. every rank solves its share of the anchors and fills the profile rows
       K(anchor, candidates of query j) of *every* query that uses them, in a
       zero-initialised [B][T+1][s] block; one all-reduce(sum) assembles the
       block (each row has exactly one non-zero contributor, so the sum is
       exact) -- the only collective on the data path, T*s doubles per query;
    4. every rank reranks its own queries; the ranked lists are gathered in
       query order.
    `engine` (tests) replaces the device engine; it must provide query_stage,
    anchor_stage, rerank_stage and the attributes T and s_eff."""
    import torch
    import torch.distributed as dist

    from .linkpred import SparseKatzEngine, sparse_katz_batch

    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    else:
        world, rank = 1, 0
    if world == 1 and engine is None:
        return sparse_katz_batch(idx, qs, s, T, tol)
    eng = engine if engine is not None else SparseKatzEngine(idx, s, T, tol)
    qs = np.atleast_1d(np.asarray(qs, dtype=np.int64))
    sizes = [int(shard(qs, world, r).size) for r in range(world)]
    mine = shard(qs, world, rank)
    state = eng.query_stage(mine) if mine.size else None
    # (2) small tables to every rank
    local = None
    if state is not None:
        local = (state["anc"].cpu().numpy(), state["top"].cpu().numpy(), state["counts"].cpu().numpy())
    if world > 1:
        tables = [None] * world
        dist.all_gather_object(tables, local, group=group)
    else:
        tables = [local]
    tables = [t for t in tables if t is not None]
    anc_all = np.concatenate([t[0] for t in tables], axis=0)
    top_all = np.concatenate([t[1] for t in tables], axis=0)
    counts_all = np.concatenate([t[2] for t in tables], axis=0)
    B = anc_all.shape[0]
    uniq, inverse = np.unique(anc_all, return_inverse=True)
    inverse = inverse.reshape(B, eng.T)
    bounds = np.linspace(0, uniq.size, world + 1).astype(np.int64)
    u0, u1 = int(bounds[rank]), int(bounds[rank + 1])
    # (3) my share of the anchors, for every query that uses them
    dev = state["profiles"].device if state is not None else ("cuda" if engine is None else "cpu")
    block = torch.zeros((B, eng.T + 1, eng.s_eff), dtype=torch.float64, device=dev)
    if u1 > u0:
        eng.anchor_stage(uniq[u0:u1], inverse, u0, torch.as_tensor(top_all, device=dev),
                         torch.as_tensor(counts_all, device=dev), block)
    if world > 1:
        dist.all_reduce(block, op=dist.ReduceOp.SUM, group=group)
    # (4) rerank my queries
    local_out = []
    if state is not None:
        q0 = sum(sizes[:rank])
        state["profiles"][:, 1:, :] = block[q0 : q0 + sizes[rank], 1:, :]
        local_out = eng.rerank_stage(state)
    return gather_in_order(local_out, world, group)
