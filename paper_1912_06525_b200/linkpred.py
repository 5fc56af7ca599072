"""Link-prediction scoring on the GPU with the reference's API.

Mirrors the scoring half of lrckatz.linkpred (linkpred.py:115-207):
``pearson``, ``katz_rank`` (masked top-s by exact Katz score) and
``sparse_katz`` (the anchor-profile Pearson rerank), plus batched variants
that run every query of a batch through one solve, one masked top-k
(K4) and, for sparse_katz, deduplicated anchor solves and the K7 rerank.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import solver


@dataclass(eq=False)
class RankedPrediction:
    """Ranked candidates (original id, score) for one query (linkpred.py:27-38)."""

    query: int
    candidates: list
    method: str


def pearson(x, y):
    """Pearson correlation; 0.0 for a constant vector, clipped to [-1, 1]
    (linkpred.py:115-133).  Scalar utility: evaluated on the host."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.ndim != 1 or x.shape != y.shape:
        raise ValueError("inputs must be equal-length vectors")
    if x.size < 2:
        raise ValueError("need at least two samples")
    xc = x - x.mean()
    yc = y - y.mean()
    sx = np.linalg.norm(xc)
    sy = np.linalg.norm(yc)
    if sx == 0.0 or sy == 0.0:
        return 0.0
    return float(np.clip((xc @ yc) / (sx * sy), -1.0, 1.0))


_TOPK_PASS = 4096  # entries per column one kz_topk_batch call returns
_RERANK_SMEM = 8192  # candidates kz_pearson_rerank orders in shared memory


def topk_device(scores, k, mask_op=None, mask_rows=None, self_ids=None):
    """K4 masked top-k over the columns of scores (cuda fp64 [b][n]).

    Returns (ids int64 [b][k], vals fp64 [b][k], counts int32 [b]) on the
    device; ids are positions in the scores' order (internal ids).  A k above
    4096 runs in passes: each continues below the last key of the previous
    one (kz_topk_args.bound_*), so any k up to n is exact."""
    torch = _lib.torch_cuda()
    lib = _lib.load()
    b, n = scores.shape
    k = int(k)
    ids = torch.empty((b, k), dtype=torch.int64, device="cuda")
    vals = torch.empty((b, k), dtype=torch.float64, device="cuda")
    # a single pass writes every count; several passes accumulate into zeros
    counts = (torch.empty if k <= _TOPK_PASS else torch.zeros)((b,), dtype=torch.int32, device="cuda")
    keep = []
    margs = {}
    if mask_op is not None and mask_rows is not None:
        arr, p = _lib.i64_array(mask_rows)
        keep.append(arr)
        margs["mask_graph"], margs["mask_rows"] = mask_op.handle.value, p
    if self_ids is not None:
        arr, p = _lib.i64_array(self_ids)
        keep.append(arr)
        margs["self_ids"] = p
    st = _lib.stream_ptr(torch)
    bval = bid = None
    for k0 in range(0, k, _TOPK_PASS):
        kk = min(_TOPK_PASS, k - k0)
        pi = ids if kk == k else torch.empty((b, kk), dtype=torch.int64, device="cuda")
        pv = vals if kk == k else torch.empty((b, kk), dtype=torch.float64, device="cuda")
        pc = counts if kk == k else torch.empty((b,), dtype=torch.int32, device="cuda")
        args = _lib.KzTopkArgs()
        args.b, args.k, args.n = b, kk, n
        args.scores = scores.data_ptr()
        for name, v in margs.items():
            setattr(args, name, v)
        args.ids_out, args.vals_out, args.count_out = pi.data_ptr(), pv.data_ptr(), pc.data_ptr()
        if bid is not None:
            args.bound_vals, args.bound_ids = bval.data_ptr(), bid.data_ptr()
        ws = _lib.Workspace.get(torch, lib.kz_topk_workspace_bytes(b, n, kk), slot="topk")
        _lib.check(lib.kz_topk_batch(ctypes.byref(args), _lib.ptr(ws), ws.numel(), st))
        if kk == k:
            break
        ids[:, k0 : k0 + kk] = pi
        vals[:, k0 : k0 + kk] = pv
        counts += pc
        # continue strictly below each column's last key; a column that came
        # up short has nothing left (its next passes return 0 entries)
        last = (pc.to(torch.int64) - 1).clamp(min=0).unsqueeze(1)
        bval = torch.gather(pv, 1, last).squeeze(1).contiguous()
        bid = torch.where(pc > 0, torch.gather(pi, 1, last).squeeze(1), torch.full_like(pc, -1, dtype=torch.int64))
        # an exhausted column must return nothing more: bound it at the
        # smallest possible key (score 0, id n-1)
        bid = torch.where(pc < kk, torch.full_like(bid, n - 1), bid).contiguous()
        bval = torch.where(pc < kk, torch.zeros_like(bval), bval).contiguous()
    return ids, vals, counts


def _query_batch_state(idx, qs, tol):
    scores, _ = solver.query_batch(idx, qs, tol=tol, device=True)
    internal = idx.internal_ids(qs)
    return scores, internal


def katz_rank_batch(idx, qs, s, tol=1e-10):
    """katz_rank for many queries: one batched solve + one masked top-s."""
    if s < 1:
        raise ValueError("s must be >= 1")
    qs = np.atleast_1d(np.asarray(qs, dtype=np.int64))
    try:
        scores, internal = _query_batch_state(idx, qs, tol)
    except KeyError as err:
        raise solver.UnknownNodeError(str(err)) from None
    s_eff = min(int(s), idx.n)
    ids, vals, counts = topk_device(scores, s_eff, idx.mask_operator(), internal, internal)
    ids, vals, counts = ids.cpu().numpy(), vals.cpu().numpy(), counts.cpu().numpy()
    orig = np.asarray(idx.id_map)[np.maximum(ids, 0)]  # internal -> original ids, one gather
    out = []
    for j, q in enumerate(qs.tolist()):
        m = int(counts[j])
        cands = list(zip(orig[j, :m].tolist(), vals[j, :m].tolist()))
        out.append(RankedPrediction(query=q, candidates=cands, method="katz"))
    return out


def katz_rank(idx, q, s, tol=1e-10):
    """Top-s predicted links for q by exact Katz score (linkpred.py:155-162)."""
    if s < 1:
        raise ValueError("s must be >= 1")
    return katz_rank_batch(idx, [q], s, tol)[0]


class SparseKatzEngine:
    """The three device stages of sparse_katz (linkpred.py:165-207) for a
    batch of queries: (1) query solves, masked top-s candidates, top-T
    anchors and the reference profiles; (2) anchor solves gathered straight
    into candidate profiles (K7 gather); (3) the Pearson rerank (K7).
    ``sparse_katz_batch`` runs them in one process; ``distributed.
    sparse_katz_distributed`` runs stage 2 on the globally deduplicated anchor
    set, sharded over the ranks."""

    def __init__(self, idx, s, T=None, tol=1e-10, anchor_batch=256):
        if s < 1:
            raise ValueError("s must be >= 1")
        if T is None:
            T = s + 1
        if T < 1:
            raise ValueError("need at least one anchor")
        if T > idx.n - 1:
            raise ValueError(f"T={T} anchors not available on {idx.n} nodes")
        self.idx, self.T, self.tol, self.anchor_batch = idx, int(T), tol, int(anchor_batch)
        self.s_eff = min(int(s), idx.n)
        self.torch = _lib.torch_cuda()

    def query_stage(self, qs):
        """-> dict(qs, top [b][s] int64, top_vals, counts [b] int32, anc [b][T]
        int64, ref [b][T+1], profiles [b][T+1][s] with row 0 filled); device
        tensors, ids internal."""
        torch, idx, T = self.torch, self.idx, self.T
        qs = np.atleast_1d(np.asarray(qs, dtype=np.int64))
        try:
            scores, internal = _query_batch_state(idx, qs, self.tol)
        except KeyError as err:
            raise solver.UnknownNodeError(str(err)) from None
        b = scores.shape[0]
        top, top_vals, counts = topk_device(scores, self.s_eff, idx.mask_operator(), internal, internal)
        anc, _, _ = topk_device(scores, T, None, None, internal)
        # reference profile [K(q,q), K(a_i,q)]  (linkpred.py:189-191)
        qidx = torch.as_tensor(internal, dtype=torch.int64, device="cuda")
        rows = torch.arange(b, device="cuda")
        ref = torch.empty((b, T + 1), dtype=torch.float64, device="cuda")
        ref[:, 0] = scores[rows, qidx]
        ref[:, 1:] = torch.gather(scores, 1, anc)
        profiles = torch.empty((b, T + 1, self.s_eff), dtype=torch.float64, device="cuda")
        profiles[:, 0, :] = top_vals
        return {"qs": qs, "top": top, "top_vals": top_vals, "counts": counts, "anc": anc, "ref": ref,
                "profiles": profiles}

    def anchor_stage(self, uniq, inverse, u0, top, counts, profiles):
        """Solve the anchors uniq (internal ids) in batches and write
        profiles[j][i+1][:] = K(anchor, top[j][:]) for every slot (j, i) with
        u0 <= inverse[j][i] < u0 + len(uniq); inverse indexes the global
        unique list whose slice [u0, u0+len(uniq)) is `uniq`."""
        torch, idx = self.torch, self.idx
        lib = _lib.load()
        st = _lib.stream_ptr(torch)
        n = idx.n
        T1 = profiles.shape[1]
        for s0 in range(0, len(uniq), self.anchor_batch):
            chunk = uniq[s0 : s0 + self.anchor_batch]
            a_scores, _ = solver.query_batch(idx, idx.id_map[chunk], tol=self.tol, device=True)
            lo = u0 + s0
            sel = np.argwhere((inverse >= lo) & (inverse < lo + chunk.size))
            trip = np.stack([inverse[sel[:, 0], sel[:, 1]] - lo, sel[:, 0], sel[:, 1] + 1], axis=1)
            trip_d = torch.as_tensor(np.ascontiguousarray(trip, dtype=np.int64), device="cuda")
            _lib.check(lib.kz_profile_gather(_lib.ptr(a_scores), n, int(trip.shape[0]), _lib.ptr(trip_d),
                                             _lib.ptr(top), _lib.ptr(counts), self.s_eff, _lib.ptr(profiles),
                                             T1, st))
            del a_scores

    def rerank_stage(self, state):
        """Pearson rerank of every query's candidates -> [RankedPrediction]."""
        torch, idx, s_eff = self.torch, self.idx, self.s_eff
        lib = _lib.load()
        st = _lib.stream_ptr(torch)
        top, top_vals, counts = state["top"], state["top_vals"], state["counts"]
        profiles, ref = state["profiles"], state["ref"]
        b, T1 = ref.shape
        corr = torch.empty((b, s_eff), dtype=torch.float64, device="cuda")
        big = s_eff > _RERANK_SMEM
        order = None if big else torch.empty((b, s_eff), dtype=torch.int64, device="cuda")
        _lib.check(lib.kz_pearson_rerank(_lib.ptr(profiles), _lib.ptr(ref), _lib.ptr(top), _lib.ptr(top_vals),
                                         _lib.ptr(counts), b, T1, s_eff, _lib.ptr(corr), _lib.ptr(order), st))
        if big:
            # more candidates than one CTA sorts in shared memory: the same
            # lexsort((top, -score, -corr)) as three stable device sorts
            valid = torch.arange(s_eff, device="cuda").unsqueeze(0) < counts.unsqueeze(1)
            key_c = torch.where(valid, -corr, torch.full_like(corr, float("inf")))
            order = torch.argsort(top, dim=1, stable=True)
            order = torch.gather(order, 1, torch.argsort(torch.gather(-top_vals, 1, order), dim=1, stable=True))
            order = torch.gather(order, 1, torch.argsort(torch.gather(key_c, 1, order), dim=1, stable=True))
        top_h, corr_h, order_h, counts_h = (top.cpu().numpy(), corr.cpu().numpy(), order.cpu().numpy(),
                                            counts.cpu().numpy())
        out = []
        for j, q in enumerate(state["qs"].tolist()):
            m = int(counts_h[j])
            o = order_h[j, :m]
            ids_j = np.asarray(idx.id_map)[top_h[j, o]]
            cands = list(zip(ids_j.tolist(), corr_h[j, o].tolist()))
            out.append(RankedPrediction(query=q, candidates=cands, method="sparse-katz"))
        return out


def sparse_katz_batch(idx, qs, s, T=None, tol=1e-10, anchor_batch=256):
    """sparse_katz for many queries (linkpred.py:165-207), batched.

    The anchor solves of all queries are deduplicated and run in batches of
    ``anchor_batch`` columns; each batch's scores are gathered straight into
    the candidates' profiles (K7 gather) and dropped, so the device holds at
    most one batch of anchor score vectors."""
    eng = SparseKatzEngine(idx, s, T, tol, anchor_batch)
    state = eng.query_stage(qs)
    b = state["anc"].shape[0]
    uniq, inverse = np.unique(state["anc"].cpu().numpy(), return_inverse=True)
    eng.anchor_stage(uniq, inverse.reshape(b, eng.T), 0, state["top"], state["counts"], state["profiles"])
    return eng.rerank_stage(state)


def sparse_katz(idx, q, s, T=None, tol=1e-10):
    """Rerank the top-s Katz candidates by anchor-profile correlation
    (linkpred.py:165-207)."""
    return sparse_katz_batch(idx, [q], s, T, tol)[0]
