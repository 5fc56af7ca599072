"""Link-prediction recall harness on the batched GPU rankers.

Mirrors the evaluation half of lrckatz.linkpred (linkpred.py:20-112,
210-337): ``temporal_split`` builds the train graph and the held-out
positive pairs (bucketed by the smaller train degree of the pair), and
``evaluate_recall`` / ``evaluate_recall_sweep`` measure recall@s of a
ranking method.  The rankings come from ``katz_rank_batch`` /
``sparse_katz_batch`` -- all queries of a run go through the device in
batches instead of one solve per Python call; the statistics are computed
exactly as the reference does (same query order, same means/stds).
"""

from __future__ import annotations

from dataclasses import dataclass

import threading

import numpy as np

from .graph import Graph, from_edges, largest_connected_component
from .linkpred import katz_rank_batch, sparse_katz_batch

BUCKET_LABELS = ("1-3", "4-10", ">10")


class EmptyPositivesError(ValueError):
    """The split left no usable positive pairs to evaluate (linkpred.py:23-24)."""


@dataclass(eq=False)
class LinkPredDataset:
    """Train graph plus held-out positive pairs (linkpred.py:41-52)."""

    train: Graph
    positives: list
    buckets: dict


@dataclass(frozen=True)
class RecallStat:
    mean: float
    std: float
    n_queries: int


def _bucket_of(min_degree):
    return "1-3" if min_degree <= 3 else ("4-10" if min_degree <= 10 else ">10")


def temporal_split(edges_with_time, cutoff):
    """Train graph (LCC of edges with t <= cutoff) and positives (later pairs
    with both endpoints in it, not train edges), semantics of
    linkpred.py:63-112."""
    rows = list(edges_with_time)
    if not rows:
        raise ValueError("no timestamped edges")
    arr = np.asarray([(int(u), int(v), float(t)) for u, v, t in rows], dtype=np.float64)
    times = arr[:, 2]
    if cutoff < times.min():
        raise ValueError("cutoff precedes every edge; train split is empty")
    train_pairs = arr[times <= cutoff][:, :2].astype(np.int64)
    test_rows = arr[times > cutoff]
    ids = np.unique(train_pairs)
    g = largest_connected_component(from_edges(np.searchsorted(ids, train_pairs), n=ids.size, original_ids=ids))
    oid = g.original_ids
    in_train = set(int(x) for x in oid)
    rows_of = np.repeat(np.arange(g.n), np.diff(g.row_offsets))
    upper = g.col_indices > rows_of
    train_edges = set(zip(oid[rows_of[upper]].tolist(), oid[g.col_indices[upper]].tolist()))
    positives, seen = [], set()
    for u, v, _ in test_rows:
        u, v = int(u), int(v)
        if u == v:
            continue
        pair = (u, v) if u < v else (v, u)
        if pair in seen or pair in train_edges:
            continue
        if pair[0] in in_train and pair[1] in in_train:
            seen.add(pair)
            positives.append(pair)
    deg = np.diff(g.row_offsets)
    buckets = {label: [] for label in BUCKET_LABELS}
    for pair in positives:
        md = min(deg[g.internal_id(pair[0])], deg[g.internal_id(pair[1])])
        buckets[_bucket_of(int(md))].append(pair)
    return LinkPredDataset(train=g, positives=positives, buckets=buckets)


def _partners(dataset):
    partners = {}
    for u, v in dataset.positives:
        partners.setdefault(u, set()).add(v)
        partners.setdefault(v, set()).add(u)
    return partners


def _pair_bucket(dataset):
    pb = {}
    for label in BUCKET_LABELS:
        for pair in dataset.buckets[label]:
            pb[tuple(pair)] = label
    return pb


def rank_lists(idx, method, queries, pool, T=None, tol=1e-10, batch=256, workers=1):
    """Ranked candidate ids (original) for every query, in query order.

    Queries are answered in blocks of `batch` (one batched device call per
    block).  With workers > 1 the blocks run on that many host threads, each
    on its own CUDA stream, over the one shared index (the reference's
    ThreadPoolExecutor fan-out, linkpred.py:309-317).  The block composition
    does not depend on `workers`, so every query's result -- and every
    statistic built from them -- is identical for any worker count."""
    def rank_block(qs):
        if method == "katz":
            preds = katz_rank_batch(idx, qs, pool, tol=tol)
        elif method == "sparse-katz":
            preds = sparse_katz_batch(idx, qs, pool, T=T, tol=tol)
        else:
            raise ValueError(f"unknown method {method!r}")
        return [[c for c, _ in p.candidates] for p in preds]

    blocks = [np.asarray(queries[s0 : s0 + batch], dtype=np.int64) for s0 in range(0, len(queries), batch)]
    if workers <= 1 or len(blocks) <= 1:
        return [lst for qs in blocks for lst in rank_block(qs)]
    from concurrent.futures import ThreadPoolExecutor

    from . import _lib

    torch = _lib.torch_cuda()
    idx.operator(), idx.mask_operator()  # create the shared device state once, up front
    local = threading.local()
    caller = torch.cuda.current_stream()

    def run(qs):
        st = getattr(local, "stream", None)
        if st is None:
            st = local.stream = torch.cuda.Stream()
        st.wait_stream(caller)
        with torch.cuda.stream(st):
            out = rank_block(qs)
        st.synchronize()
        return out

    with ThreadPoolExecutor(max_workers=workers) as ex:
        return [lst for res in ex.map(run, blocks) for lst in res]


def _stat(recalls):
    if not recalls:
        return RecallStat(float("nan"), float("nan"), 0)
    arr = np.asarray(recalls)
    return RecallStat(float(arr.mean()), float(arr.std()), len(recalls))


def evaluate_recall(idx, method, dataset, s, T=None, query_sample=None, pool=None, tol=1e-10):
    """Mean recall@s over the held-out positives (linkpred.py:238-279)."""
    if not dataset.positives:
        raise EmptyPositivesError("no positive pairs to evaluate")
    partners = _partners(dataset)
    queries = sorted(partners) if query_sample is None else sorted(query_sample)
    for u in queries:
        if u not in partners:
            raise ValueError(f"query {u} has no positive partners")
    if not queries:
        raise EmptyPositivesError("query sample is empty")
    pb = _pair_bucket(dataset)
    fetch = max(pool, s) if pool is not None else s
    ranked = rank_lists(idx, method, queries, fetch, T, tol)
    per = {label: [] for label in ("overall", *BUCKET_LABELS)}
    for u, lst in zip(queries, ranked):
        top = set(lst[:s])
        mine = partners[u]
        per["overall"].append(len(top & mine) / len(mine))
        for label in BUCKET_LABELS:
            inb = {v for v in mine if pb[(u, v) if u < v else (v, u)] == label}
            if inb:
                per[label].append(len(top & inb) / len(inb))
    return {label: _stat(r) for label, r in per.items()}


def evaluate_recall_sweep(idx, methods, dataset, s_values, T=None, query_sample=None, tol=1e-10, workers=1,
                          batch=256):
    """Recall@s for several methods and sizes from one ranking per query
    (linkpred.py:282-337).  `workers` > 1 answers the query blocks on that
    many threads and CUDA streams (rank_lists); the statistics do not depend
    on it (reference tests/test_linkpred.py:355-365)."""
    if not dataset.positives:
        raise EmptyPositivesError("no positive pairs to evaluate")
    s_values = sorted(set(int(s) for s in s_values))
    pool = s_values[-1]
    partners = _partners(dataset)
    queries = sorted(partners) if query_sample is None else sorted(query_sample)
    if not queries:
        raise EmptyPositivesError("query sample is empty")
    pb = _pair_bucket(dataset)
    rows = []
    for method in methods:
        per = {(label, s): [] for label in ("overall", *BUCKET_LABELS) for s in s_values}
        ranked = rank_lists(idx, method, queries, pool, T, tol, batch=batch, workers=workers)
        for u, lst in zip(queries, ranked):
            mine = partners[u]
            by_label = {label: {v for v in mine if pb[(u, v) if u < v else (v, u)] == label}
                        for label in BUCKET_LABELS}
            for s in s_values:
                top = set(lst[:s])
                per[("overall", s)].append(len(top & mine) / len(mine))
                for label in BUCKET_LABELS:
                    if by_label[label]:
                        per[(label, s)].append(len(top & by_label[label]) / len(by_label[label]))
        for (label, s), recalls in sorted(per.items()):
            rows.append((method, label, s, _stat(recalls)))
    return rows
