"""world_size-2 gloo test of the query-column sharding and result gather
(CPU): each rank ranks its shard with the oracle and the gathered result
must equal the single-process answer in query order."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_rank(qs):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import katz_oracle as O

    rec = np.load(os.path.join(GOLDEN, "chunglu2000_cg.npz"))
    n = rec["row_offsets"].size - 1
    a = O.csr_matrix(rec["row_offsets"], rec["col_indices"], n)
    beta = float(rec["beta"])
    solve = lambda i: O.query_cg_csr(a, beta, i, tol=1e-10)[0]  # noqa: E731
    nbrs = lambda i: a.indices[a.indptr[i] : a.indptr[i + 1]]  # noqa: E731
    return [O.katz_rank(solve, nbrs, np.arange(n), int(q), 5) for q in qs]


def _worker(rank, world, port, qs, out):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1912_06525_b200.distributed import shard, sharded

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    assert shard(qs, world, rank).size in (len(qs) // world, len(qs) // world + 1)
    res = sharded(_oracle_rank, qs)
    out[rank] = res
    dist.destroy_process_group()


def test_sharded_katz_rank_gloo_world2():
    qs = np.array([3, 17, 250, 999, 1500, 1700, 42])
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), qs, out), nprocs=2, join=True)
    want = _oracle_rank(qs)
    assert out[0] == want and out[1] == want


def test_shard_covers_everything():
    from paper_1912_06525_b200.distributed import shard

    qs = np.arange(10)
    for world in (1, 2, 3, 4, 8):
        parts = [shard(qs, world, r) for r in range(world)]
        assert np.array_equal(np.concatenate(parts), qs)


class _OracleSparseKatzEngine:
    """Host stand-in for linkpred.SparseKatzEngine (same three stages, numpy +
    the oracle's CG) so the exchange protocol of sparse_katz_distributed runs
    on CPU ranks."""

    def __init__(self, s, T=None, tol=1e-10):
        import sys

        sys.path.insert(0, ROOT)
        from oracle import katz_oracle as O

        rec = np.load(os.path.join(GOLDEN, "chunglu2000_cg.npz"))
        self.O = O
        self.n = rec["row_offsets"].size - 1
        self.a = O.csr_matrix(rec["row_offsets"], rec["col_indices"], self.n)
        self.beta = float(rec["beta"])
        self.tol = tol
        self.s_eff = min(s, self.n)
        self.T = s + 1 if T is None else T
        self.solves = 0

    def solve(self, i):
        self.solves += 1
        return self.O.query_cg_csr(self.a, self.beta, int(i), tol=self.tol)[0]

    def nbrs(self, i):
        return self.a.indices[self.a.indptr[i] : self.a.indptr[i + 1]]

    def query_stage(self, qs):
        import torch

        b, n, s, T = len(qs), self.n, self.s_eff, self.T
        top = np.zeros((b, s), dtype=np.int64)
        counts = np.zeros(b, dtype=np.int32)
        anc = np.zeros((b, T), dtype=np.int64)
        ref = np.zeros((b, T + 1))
        prof = np.zeros((b, T + 1, s))
        self.scores = {}
        for j, q in enumerate(qs):
            q = int(q)
            sc = self.solve(q)
            self.scores[q] = sc
            t = self.O.candidate_order(n, sc, q, self.nbrs(q), s)
            counts[j] = t.size
            top[j, : t.size] = t
            order = np.lexsort((np.arange(n), -sc))
            anc[j] = [x for x in order if x != q][:T]
            ref[j, 0] = sc[q]
            ref[j, 1:] = sc[anc[j]]
            prof[j, 0, : t.size] = sc[t]
        return {"qs": np.asarray(qs, dtype=np.int64), "top": torch.from_numpy(top), "top_vals": None,
                "counts": torch.from_numpy(counts), "anc": torch.from_numpy(anc), "ref": torch.from_numpy(ref),
                "profiles": torch.from_numpy(prof)}

    def anchor_stage(self, uniq, inverse, u0, top, counts, profiles):
        for k, anchor in enumerate(uniq):
            sc = self.solve(anchor)
            for j, i in np.argwhere(inverse == u0 + k):
                m = int(counts[j])
                profiles[j, i + 1, :m] = profiles.new_tensor(sc[top[j, :m].numpy()])

    def rerank_stage(self, state):
        out = []
        for j, q in enumerate(state["qs"].tolist()):
            m = int(state["counts"][j])
            top = state["top"][j, :m].numpy()
            if m == 0:
                out.append([])
                continue
            ref = state["ref"][j].numpy()
            profiles = state["profiles"][j, :, :m].numpy()
            sc = self.scores[q]
            ref_c = ref - ref.mean()
            sr = np.linalg.norm(ref_c)
            pc = profiles - profiles.mean(axis=0)
            sp_ = np.linalg.norm(pc, axis=0)
            corr = np.zeros(m)
            ok = (sp_ > 0.0) & (sr > 0.0)
            if sr > 0.0:
                corr[ok] = np.clip((ref_c @ pc[:, ok]) / (sr * sp_[ok]), -1.0, 1.0)
            rr = np.lexsort((top, -sc[top], -corr))
            out.append([(int(top[i]), float(corr[i])) for i in rr])
        return out


def _sk_worker(rank, world, port, qs, s, out):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1912_06525_b200.distributed import sparse_katz_distributed

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    eng = _OracleSparseKatzEngine(s)
    res = sparse_katz_distributed(None, qs, s, engine=eng)
    out[rank] = (res, eng.solves)
    dist.destroy_process_group()


def test_sparse_katz_distributed_dedupes_anchors_gloo_world2():
    """Stage exchange of sparse_katz_distributed on two gloo ranks: results
    equal the single-process oracle's sparse_katz for every query, and the
    ranks together solve each distinct anchor once."""
    s = 4
    qs = np.array([3, 17, 250, 999, 1500])
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_sk_worker, args=(2, _free_port(), qs, s, out), nprocs=2, join=True)
    eng = _OracleSparseKatzEngine(s)
    O = eng.O
    want = [O.sparse_katz(eng.solve, eng.nbrs, np.arange(eng.n), int(q), s) for q in qs]
    anchors = set()
    for q in qs:
        sc = eng.solve(int(q))
        order = np.lexsort((np.arange(eng.n), -sc))
        anchors.update([int(x) for x in order if x != q][: s + 1])
    for r in (0, 1):
        got = out[r][0]
        assert len(got) == len(want)
        for g, w in zip(got, want):
            assert [c for c, _ in g] == [c for c, _ in w]
            assert np.allclose([v for _, v in g], [v for _, v in w], rtol=0, atol=1e-12)
    assert out[0][1] + out[1][1] == len(qs) + len(anchors) < len(qs) * (s + 2)
