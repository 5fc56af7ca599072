"""GPU parity of K1 (SpMM), K2 (batched CG) and K4 (top-k) against the oracle.

Tolerances (BASELINE.json north_star): scores within relative L2 1e-10 per
query column, CG iteration counts within +/-1 of the same-recurrence CPU
oracle; top-k identical apart from ties within tolerance.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import katz_oracle as O

pytestmark = pytest.mark.gpu

REL_TOL = 1e-10


@pytest.fixture(scope="module")
def torch():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def kz(torch):
    import paper_1912_06525_b200 as kz

    return kz


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def chunglu_fixture():
    rec = np.load(os.path.join(GOLDEN, "chunglu2000_cg.npz"))
    n = rec["row_offsets"].size - 1
    return rec, n


def to_blk(X, C):
    """[n][b] -> chunked [b/C][n][C]"""
    n, b = X.shape
    return np.ascontiguousarray(X.T.reshape(b // C, C, n).transpose(0, 2, 1))


def from_blk(Y, n, b, C):
    return Y.reshape(b // C, n, C).transpose(0, 2, 1).reshape(b, n).T


@pytest.mark.parametrize("graph", ["chunglu2000", "rmat12"])
@pytest.mark.parametrize("b,C", [(1, 1), (4, 4), (16, 16), (32, 16), (32, 32), (8, 2)])
def test_spmm_matches_scipy(torch, kz, graph, b, C):
    if graph == "chunglu2000":
        rec, n = chunglu_fixture()
        off, col = rec["row_offsets"], rec["col_indices"]
    else:
        from paper_1912_06525_b200.generators import rmat_graph

        g = rmat_graph(12, seed=3)
        n, off, col = g.n, g.row_offsets, g.col_indices
    a = O.csr_matrix(off, col, n)
    op = kz.DeviceOperator(off, col.astype(np.int32), n)
    rng = np.random.default_rng(b * 100 + C)
    X = rng.standard_normal((n, b))
    beta = 0.013
    Xd = torch.as_tensor(to_blk(X, C)).cuda()
    Yd = torch.empty_like(Xd)
    dots = torch.empty(b, dtype=torch.float64, device="cuda")
    op.spmm(Xd, Yd, b=b, chunk=C, Xs=Xd, s1=1.0, s2=-beta, dots=dots)
    Y = from_blk(Yd.cpu().numpy(), n, b, C)
    want = X - beta * (a @ X)
    split_rows = np.diff(off) > 32
    # short rows (one lane group each) sum in CSR order with the same
    # roundings as scipy: bit-exact; warp-split rows differ by roundoff only
    assert np.array_equal(Y[~split_rows], want[~split_rows])
    assert np.abs(Y - want).max() <= 1e-13 * np.abs(want).max()
    want_dots = np.einsum("ij,ij->j", X, want)
    assert np.allclose(dots.cpu().numpy(), want_dots, rtol=1e-12, atol=0)
    # deterministic: a second launch is bit-identical
    Y2 = torch.empty_like(Xd)
    op.spmm(Xd, Y2, b=b, chunk=C, Xs=Xd, s1=1.0, s2=-beta)
    assert torch.equal(Yd, Y2)


def test_spmm_chunk64_products_and_dot_guard(torch, kz):
    """Chunk width 64 (512-byte rows) is a valid K1 width for the product;
    the fused column dots map one lane to one column of a chunk, so they are
    refused above 32 with a clear error instead of returning partial dots."""
    rec, n = chunglu_fixture()
    off, col = rec["row_offsets"], rec["col_indices"]
    a = O.csr_matrix(off, col, n)
    op = kz.DeviceOperator(off, col.astype(np.int32), n)
    X = np.random.default_rng(64).standard_normal((n, 64))
    Xd = torch.as_tensor(to_blk(X, 64)).cuda()
    Yd = torch.empty_like(Xd)
    op.spmm(Xd, Yd, b=64, chunk=64, Xs=Xd, s1=1.0, s2=-0.013)
    want = X - 0.013 * (a @ X)
    assert np.abs(from_blk(Yd.cpu().numpy(), n, 64, 64) - want).max() <= 1e-13 * np.abs(want).max()
    dots = torch.empty(64, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="chunk width of at most 32"):
        op.spmm(Xd, Yd, b=64, chunk=64, Xs=Xd, s1=1.0, s2=-0.013, dots=dots)


@pytest.mark.parametrize("slice_mb,min_deg", [(0.002, 40), (0.01, 128), (0.002, 1024)])
def test_spmm_column_blocked_schedule(torch, kz, monkeypatch, slice_mb, min_deg):
    """The opt-in column-blocked long-row schedule of K1 (graph.cu SchedOpts,
    forced here by a tiny KZ_K1_SLICE_MB): same operator, short rows still
    bit-exact against scipy, the rest within roundoff, deterministic."""
    from paper_1912_06525_b200.generators import rmat_graph

    g = rmat_graph(12, seed=3)
    n, off, col = g.n, g.row_offsets, g.col_indices
    a = O.csr_matrix(off, col, n)
    monkeypatch.setenv("KZ_K1_SLICE_MB", str(slice_mb))
    monkeypatch.setenv("KZ_K1_MINDEG", str(min_deg))
    op = kz.DeviceOperator(off, col.astype(np.int32), n)
    monkeypatch.delenv("KZ_K1_SLICE_MB")
    b, C = 32, 32
    X = np.random.default_rng(5).standard_normal((n, b))
    Xd = torch.as_tensor(to_blk(X, C)).cuda()
    Yd = torch.empty_like(Xd)
    dots = torch.empty(b, dtype=torch.float64, device="cuda")
    op.spmm(Xd, Yd, b=b, chunk=C, Xs=Xd, s1=1.0, s2=-0.01, dots=dots)
    Y = from_blk(Yd.cpu().numpy(), n, b, C)
    want = X - 0.01 * (a @ X)
    short = np.diff(off) <= 32
    assert np.array_equal(Y[short], want[short])
    assert np.abs(Y - want).max() <= 1e-13 * np.abs(want).max()
    assert np.allclose(dots.cpu().numpy(), np.einsum("ij,ij->j", X, want), rtol=1e-12, atol=0)
    Y2 = torch.empty_like(Xd)
    op.spmm(Xd, Y2, b=b, chunk=C, Xs=Xd, s1=1.0, s2=-0.01)
    assert torch.equal(Yd, Y2)


def test_cg_batch_matches_reference_cg_golden(torch, kz):
    rec, n = chunglu_fixture()
    g = kz.Graph(n=n, row_offsets=rec["row_offsets"], col_indices=rec["col_indices"],
                 original_ids=np.arange(n))
    idx = kz.GraphIndex(g, float(rec["beta"]))
    scores, reps = kz.query_cg_baseline_batch(idx, rec["queries"], tol=1e-8)
    for j in range(len(rec["queries"])):
        assert abs(reps[j].iterations - rec["iters"][j]) <= 1
        assert reps[j].converged
        assert rel(scores[j], rec["scores"][j]) <= REL_TOL
        assert reps[j].final_residual_norm == pytest.approx(rec["resid"][j], rel=1e-6)


def test_spectral_norm_matches_reference(torch, kz):
    rec, n = chunglu_fixture()
    g = kz.Graph(n=n, row_offsets=rec["row_offsets"], col_indices=rec["col_indices"],
                 original_ids=np.arange(n))
    lam = kz.spectral_norm(g)
    assert lam == pytest.approx(float(rec["spectral_norm"]), rel=1e-9)


NAMES = ["k2", "p4", "p5split", "star5", "triangle", "er40", "er60", "ba300", "ba1200"]


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("tol", [1e-8, 1e-10])
def test_query_cg_baseline_on_klrc_matches_reference(torch, kz, name, tol):
    idx = kz.load_index(os.path.join(GOLDEN, f"{name}.klrc"))
    rec = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    key = f"cg_{tol:.0e}"
    scores, reps = kz.query_cg_baseline_batch(idx, rec["queries"], tol=tol)
    for j in range(len(rec["queries"])):
        assert abs(reps[j].iterations - rec[f"{key}_iters"][j]) <= 1
        assert rel(scores[j], rec[f"{key}_scores"][j]) <= REL_TOL
        assert reps[j].converged == bool(rec[f"{key}_conv"][j])
    # single-query drop-in path
    kv, rep = kz.query_cg_baseline(idx, int(rec["queries"][0]), tol=tol)
    assert kv.scores.shape == (idx.n,) and kv.query == int(rec["queries"][0]) and kv.alpha == idx.alpha
    assert rel(kv.scores, rec[f"{key}_scores"][0]) <= REL_TOL


@pytest.mark.parametrize("name", ["er40", "ba300", "ba1200"])
def test_cg_seeded_start_and_budget(torch, kz, name):
    idx = kz.load_index(os.path.join(GOLDEN, f"{name}.klrc"))
    rec = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    q0 = int(rec["queries"][0])
    kv, rep = kz.query_cg_baseline(idx, q0, tol=1e-10, start_seed=5)
    assert abs(rep.iterations - int(rec["cg_seed5_iters"])) <= 1
    assert rel(kv.scores, rec["cg_seed5_scores"]) <= REL_TOL
    kv, rep = kz.query_cg_baseline(idx, q0, tol=1e-12, max_iter=1)
    assert rep.iterations == 1 and rep.converged == bool(rec["cg_budget1_conv"])
    assert rel(kv.scores, rec["cg_budget1_scores"]) <= REL_TOL


def test_unknown_node_and_not_spd(torch, kz):
    idx = kz.load_index(os.path.join(GOLDEN, "er40.klrc"))
    with pytest.raises(kz.UnknownNodeError):
        kz.query_cg_baseline(idx, 10**9)
    rec, n = chunglu_fixture()
    g = kz.Graph(n=n, row_offsets=rec["row_offsets"], col_indices=rec["col_indices"],
                 original_ids=np.arange(n))
    bad = kz.GraphIndex(g, 5.0 / float(rec["spectral_norm"]))  # I - 5A/lambda is indefinite
    with pytest.raises(RuntimeError):
        kz.query_cg_baseline_batch(bad, rec["queries"], tol=1e-12)


def test_generic_cg_matches_direct_solve(torch, kz):
    # tests/test_solver.py:32-58 on the device path
    b = np.random.default_rng(0).standard_normal(30)
    x, rep = kz.cg(lambda v: v, b)
    assert rep.iterations == 1 and rep.converged and np.abs(x - b).max() < 1e-14
    x, rep = kz.cg(lambda v: 2.0 * v, np.zeros(7))
    assert rep.iterations == 0 and rep.converged and np.all(x == 0.0)
    rng = np.random.default_rng(1)
    q, _ = np.linalg.qr(rng.standard_normal((50, 50)))
    a = (q * rng.uniform(0.5, 4.0, 50)) @ q.T
    b = rng.standard_normal(50)
    x, rep = kz.cg(lambda v: a @ v, b, tol=1e-10)
    assert rep.converged and rel(x, np.linalg.solve(a, b)) < 1e-8
    with pytest.raises(RuntimeError):
        kz.cg(lambda v: -v, np.ones(4))


def test_cg_katz_operator_single_call(torch, kz):
    rec, n = chunglu_fixture()
    op = kz.DeviceOperator(rec["row_offsets"], rec["col_indices"].astype(np.int32), n)
    beta = float(rec["beta"])
    q = int(rec["queries"][0])
    rhs = np.zeros(n)
    rhs[rec["col_indices"][rec["row_offsets"][q] : rec["row_offsets"][q + 1]]] = beta
    x, rep = kz.cg(kz.KatzOperator(op, beta), rhs, tol=1e-8)
    assert abs(rep.iterations - rec["iters"][0]) <= 1
    assert rel(np.maximum(x, 0), rec["scores"][0]) <= REL_TOL


@pytest.mark.parametrize("cfg", ["cfg1", "proxy16"])
def test_cg_batch_at_config_sizes(torch, kz, cfg):
    """cfg1 (Chung-Lu 10k, b=16) and the R-MAT-16 proxy (b=64) against the
    CSR oracle on a sample of columns."""
    from paper_1912_06525_b200.generators import CONFIGS, config_graph, sample_queries

    g = config_graph(cfg)
    lam = kz.spectral_norm(g)
    beta = 0.5 / lam
    idx = kz.GraphIndex(g, beta)
    b = CONFIGS[cfg]["b"]
    qs = sample_queries(g.original_ids, b, seed=0)
    scores, reps = kz.query_cg_baseline_batch(idx, qs, tol=1e-8, device=True)
    a = O.csr_matrix(g.row_offsets, g.col_indices, g.n)
    for j in np.linspace(0, b - 1, 6).astype(int):
        want, orep = O.query_cg_csr(a, beta, g.internal_id(int(qs[j])), tol=1e-8)
        assert abs(reps[j].iterations - orep.iterations) <= 1
        assert rel(scores[j].cpu().numpy(), want) <= REL_TOL


@pytest.mark.parametrize("cfg", ["cfg1", "proxy16"])
def test_cg_sparse_first_iteration_matches_dense(torch, kz, cfg, monkeypatch):
    """The first CG iteration from zero runs on the 2-walk counts instead of
    the SpMM (cg.cu, cg_sparse_pq_kernel): same iterates up to the roundings
    of q0's neighbour sums -- identical iteration counts, scores within
    1e-12 -- and run-to-run bit-identical."""
    from paper_1912_06525_b200.generators import CONFIGS, config_graph, sample_queries

    g = config_graph(cfg)
    lam = kz.spectral_norm(g)
    idx = kz.GraphIndex(g, 0.5 / lam)
    qs = sample_queries(g.original_ids, CONFIGS[cfg]["b"], seed=1)
    s1, r1 = kz.query_cg_baseline_batch(idx, qs, tol=1e-10, device=True)
    s1b, _ = kz.query_cg_baseline_batch(idx, qs, tol=1e-10, device=True)
    assert torch.equal(s1, s1b)
    monkeypatch.setenv("KZ_CG_SPARSE_FIRST", "0")
    s0, r0 = kz.query_cg_baseline_batch(idx, qs, tol=1e-10, device=True)
    monkeypatch.delenv("KZ_CG_SPARSE_FIRST")
    assert [r.iterations for r in r1] == [r.iterations for r in r0]
    diff = (torch.linalg.vector_norm(s1 - s0, dim=1) / torch.linalg.vector_norm(s0, dim=1)).cpu().numpy()
    assert np.all(diff <= 1e-12), diff.max()


@pytest.mark.parametrize("tol,slots", [(1e-8, None), (1e-12, None), (1e-12, 8), (1e-12, 4), (1e-8, 3)])
def test_cg_residual_history_matches_per_iteration_update(torch, kz, monkeypatch, tol, slots):
    """The residual-history form of the solution (x = x0 + sum c_i r_i,
    blockops.cuh CgHistory; folded into x when a solve outgrows its slots,
    which 8 / 4 / 3 slots force -- the default is up to 16) against the
    per-iteration x update (KZ_CG_HISTORY=0): identical iteration counts,
    scores within roundoff, for plain CG and the eigen form."""
    from paper_1912_06525_b200.generators import CONFIGS, config_graph, sample_queries

    g = config_graph("proxy16")
    lam = kz.spectral_norm(g)
    gi = kz.GraphIndex(g, 0.5 / lam)
    ei = kz.EigenIndex(gi, 16)
    qs = sample_queries(g.original_ids, 40, seed=2)
    for fn, idx in ((kz.query_cg_baseline_batch, gi), (kz.query_batch, ei)):
        if slots is not None:
            monkeypatch.setenv("KZ_CG_HISTORY", str(slots))
        s1, r1 = fn(idx, qs, tol=tol, device=True)
        monkeypatch.setenv("KZ_CG_HISTORY", "0")
        s0, r0 = fn(idx, qs, tol=tol, device=True)
        monkeypatch.delenv("KZ_CG_HISTORY")
        assert [r.iterations for r in r1] == [r.iterations for r in r0]
        diff = (torch.linalg.vector_norm(s1 - s0, dim=1) / torch.linalg.vector_norm(s0, dim=1)).cpu().numpy()
        assert np.all(diff <= 1e-13), diff.max()


@pytest.mark.parametrize("n", [50_000, 70_000])  # one-CTA-per-column path (n <= 65,536) and the sliced path
def test_topk_matches_lexsort(torch, kz, n):
    rng = np.random.default_rng(4)
    b = 7
    S = np.abs(rng.standard_normal((b, n)))
    S[:, ::7] = np.round(S[:, ::7], 1)  # many exact ties
    S[1, :] = 0.25  # all tied
    S[2, : n // 2] = 0.0
    Sd = torch.as_tensor(S).cuda()
    self_ids = np.array([3, 10, 0, n - 1, 5, 6, 7])
    for k in (1, 20, 100, 1000):
        ids, vals, counts = kz.topk_device(Sd, k, None, None, self_ids)
        ids, vals = ids.cpu().numpy(), vals.cpu().numpy()
        for j in range(b):
            cand = np.array([i for i in range(n) if i != self_ids[j]])
            order = cand[np.lexsort((cand, -S[j][cand]))][:k]
            assert list(ids[j]) == list(order)
            assert np.array_equal(vals[j], S[j][order])


def test_topk_masks_neighbours(torch, kz):
    rec, n = chunglu_fixture()
    op = kz.DeviceOperator(rec["row_offsets"], rec["col_indices"].astype(np.int32), n)
    S = rec["scores"]
    qs = rec["queries"]
    Sd = torch.as_tensor(S).cuda()
    for k in (5, 50, n):
        ids, vals, counts = kz.topk_device(Sd, min(k, n), op, qs, qs)
        ids, counts = ids.cpu().numpy(), counts.cpu().numpy()
        for j, q in enumerate(qs):
            nbrs = rec["col_indices"][rec["row_offsets"][q] : rec["row_offsets"][q + 1]]
            want = O.candidate_order(n, S[j], int(q), nbrs, min(k, n))
            assert counts[j] == len(want)
            assert list(ids[j][: counts[j]]) == list(want)


def test_katz_rank_graph_index_matches_oracle(torch, kz):
    rec, n = chunglu_fixture()
    g = kz.Graph(n=n, row_offsets=rec["row_offsets"], col_indices=rec["col_indices"],
                 original_ids=np.arange(n))
    beta = float(rec["beta"])
    idx = kz.GraphIndex(g, beta)
    a = O.csr_matrix(rec["row_offsets"], rec["col_indices"], n)
    solve = lambda i: O.query_cg_csr(a, beta, i, tol=1e-10)[0]  # noqa: E731
    nbrs = lambda i: a.indices[a.indptr[i] : a.indptr[i + 1]]  # noqa: E731
    preds = kz.katz_rank_batch(idx, rec["queries"][:4], 20)
    for j, q in enumerate(rec["queries"][:4]):
        want = O.katz_rank(solve, nbrs, np.arange(n), int(q), 20)
        got = preds[j].candidates
        assert [c for c, _ in got] == [c for c, _ in want]
        assert np.allclose([v for _, v in got], [v for _, v in want], rtol=1e-9, atol=0)


def test_operator_rejects_out_of_range_columns(torch, kz):
    off = np.array([0, 1, 2], dtype=np.int64)
    with pytest.raises(ValueError):
        kz.DeviceOperator(off, np.array([1, 2], dtype=np.int32), 2)  # column 2 of a 2-column operator
    with pytest.raises(ValueError):
        kz.DeviceOperator(off, np.array([1, -1], dtype=np.int32), 2)


@pytest.mark.parametrize("mode", ["1", "0"])
def test_graph_replayed_loops_match(kz, mode):
    """Both iteration drivers (driver.cuh) give the reference's CG and LRC
    answers: the device-driven graph loop (conditional WHILE node, the
    default for small solves; KZ_GRAPHS=1 forces it) and the host-driven
    loop (KZ_GRAPHS=0), each run twice to exercise the cached graph."""
    import subprocess
    import sys

    code = r'''
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1912_06525_b200 as kz
idx = kz.load_index("tests/golden/ba300.klrc")
rec = np.load("tests/golden/ba300.npz")
q = rec["queries"]
for fn, key in ((kz.query_cg_baseline_batch, "cg"), (kz.query_batch, "lrc")) * 2:
    s, r = fn(idx, q, tol=1e-10)
    for j in range(len(q)):
        want = rec[f"{key}_1e-10_scores"][j]
        assert np.linalg.norm(s[j] - want) <= 1e-10 * np.linalg.norm(want), (key, j)
        assert abs(r[j].iterations - rec[f"{key}_1e-10_iters"][j]) <= 1
print("graphs ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, KZ_GRAPHS=mode)
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True)
    assert out.returncode == 0 and "graphs ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("n", [20_000, 70_000])
def test_topk_above_one_pass_matches_lexsort(torch, kz, n):
    """k beyond one kz_topk_batch pass (4,096 per column): the continuation
    passes (bound_vals / bound_ids) give exactly np.lexsort's order,
    including heavy ties across pass boundaries and columns with fewer
    unmasked entries than k."""
    rng = np.random.default_rng(9)
    b = 3
    S = np.abs(rng.standard_normal((b, n)))
    S[0, ::3] = 0.5  # ties that straddle the 4,096 boundaries
    S[2, : n - 5000] = 0.0  # long run of equal zeros
    Sd = torch.as_tensor(S).cuda()
    self_ids = np.array([1, 2, 3])
    for k in (4096, 4097, 9000, n - 1, n + 10):
        ids, vals, counts = kz.topk_device(Sd, k, None, None, self_ids)
        ids, vals, counts = ids.cpu().numpy(), vals.cpu().numpy(), counts.cpu().numpy()
        for j in range(b):
            cand = np.array([i for i in range(n) if i != self_ids[j]])
            order = cand[np.lexsort((cand, -S[j][cand]))][:k]
            assert counts[j] == len(order)
            assert np.array_equal(ids[j][: len(order)], order)
            assert np.array_equal(vals[j][: len(order)], S[j][order])
            assert np.all(ids[j][len(order):] == -1)


def test_katz_rank_with_s_above_one_topk_pass(torch, kz):
    """katz_rank with s > 4,096 candidates equals the oracle's
    _candidate_order (linkpred.py:145-152) at full length."""
    rec, n = chunglu_fixture()
    g = kz.Graph(n=n, row_offsets=rec["row_offsets"], col_indices=rec["col_indices"], original_ids=np.arange(n))
    beta = float(rec["beta"])
    idx = kz.GraphIndex(g, beta)
    a = O.csr_matrix(rec["row_offsets"], rec["col_indices"], n)
    q = int(rec["queries"][0])
    s = n  # every candidate
    pred = kz.katz_rank_batch(idx, [q], s, tol=1e-12)[0]
    x, _ = O.query_cg_csr(a, beta, q, tol=1e-12)
    want = O.candidate_order(n, x, q, a.indices[a.indptr[q] : a.indptr[q + 1]], s)
    got = np.array([c for c, _ in pred.candidates])
    assert len(got) == len(want)
    nx = np.linalg.norm(x)
    diff = np.flatnonzero(got != want)
    assert np.all(np.abs(x[got[diff]] - x[want[diff]]) <= 1e-12 * nx)


def test_sparse_katz_rerank_device_sort_fallback(torch, kz, monkeypatch):
    """Above 8,192 candidates the rerank order comes from stable device sorts
    instead of the shared-memory bitonic sort; both give the same
    lexsort((top, -score, -corr)) order (forced here on a small case)."""
    from paper_1912_06525_b200 import linkpred

    idx = kz.load_index(os.path.join(GOLDEN, "ba300.klrc"))
    qs = idx.id_map[::11][:8]
    want = [p.candidates for p in kz.sparse_katz_batch(idx, qs, 40)]
    monkeypatch.setattr(linkpred, "_RERANK_SMEM", 4)
    got = [p.candidates for p in kz.sparse_katz_batch(idx, qs, 40)]
    assert got == want


def test_sparse_katz_distributed_single_rank_equals_batch(torch, kz):
    """The staged path of sparse_katz_distributed (query stage, anchor stage
    over the globally deduplicated anchors, rerank stage) on one rank gives
    sparse_katz_batch's lists; the world-2 exchange is covered on gloo
    (tests/test_distributed.py)."""
    from paper_1912_06525_b200.distributed import sparse_katz_distributed
    from paper_1912_06525_b200.linkpred import SparseKatzEngine

    idx = kz.load_index(os.path.join(GOLDEN, "ba300.klrc"))
    qs = idx.id_map[::13][:10]
    want = [p.candidates for p in kz.sparse_katz_batch(idx, qs, 12)]
    got = [p.candidates for p in sparse_katz_distributed(idx, qs, 12, engine=SparseKatzEngine(idx, 12))]
    assert got == want


def test_fused_small_cg_last_column_keeps_its_final_update(kz):
    """Regression (found by tools/fuzz_parity.py): 70 queries on a 30,000-node
    path-with-chords graph, three chunks, one column of the last chunk iterating
    once more than every other.  The fused small-solve kernel rewrote its chunk
    flags while slower warps had not yet applied that chunk's last x update, so
    rows of that column missed it (rel. error ~tol with matching residuals).
    Every column must match the oracle to 1e-10 with identical iterations."""
    from paper_1912_06525_b200.graph import Graph

    z = np.load(os.path.join(GOLDEN, "fuzz_small_cg_case.npz"))
    n = z["row_offsets"].size - 1
    g = Graph(n=n, row_offsets=z["row_offsets"], col_indices=z["col_indices"].astype(np.int64),
              original_ids=z["original_ids"])
    beta, tol = float(z["beta"]), float(z["tol"])
    idx = kz.GraphIndex(g, beta, spectral_norm=float(z["lam"]), reorder=str(z["reorder"]))
    qs = z["queries"]
    am = O.csr_matrix(z["row_offsets"], z["col_indices"], n)
    internal = idx.internal_ids(qs)
    for _ in range(3):  # the race was timing dependent
        scores, reps = kz.query_cg_baseline_batch(idx, qs, tol=tol)
        scores = np.asarray(scores)
        for j in range(len(qs)):
            want, wrep = O.query_cg_csr(am, beta, int(internal[j]), tol=tol)
            assert reps[j].iterations == wrep.iterations
            assert np.linalg.norm(scores[j] - want) <= 1e-10 * np.linalg.norm(want), j


def test_vec_op_rounds_like_numpy(torch, kz):
    """kz_vec_op (the generic cg() updates) rounds the products and the sum
    separately, as numpy's x += a*p, r -= a*q, p = r + b*p do."""
    from paper_1912_06525_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(3)
    n = 100_003
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    a, b = 0.3721931, -1.77e-3
    xt, yt = torch.as_tensor(x).cuda(), torch.as_tensor(y).cuda()
    out = torch.empty_like(xt)
    _lib.vec_op(torch, lib, 0, n, a, xt, 1.0, yt, out)
    assert np.array_equal(out.cpu().numpy(), y + a * x)
    _lib.vec_op(torch, lib, 0, n, -a, xt, 1.0, yt, out)
    assert np.array_equal(out.cpu().numpy(), y - a * x)
    _lib.vec_op(torch, lib, 0, n, b, xt, 1.0, yt, out)
    assert np.array_equal(out.cpu().numpy(), y + b * x)
    _lib.vec_op(torch, lib, 1, n, 7.25, xt, 0.0, None, out)
    assert np.array_equal(out.cpu().numpy(), x / 7.25)


def test_repeated_launches_are_bit_identical(torch, kz):
    """Stand-in for racecheck (compute-sanitizer is not available on the GPU
    pool): every kernel family with cross-warp / cross-CTA reductions or
    spin-waits -- K1's last-finisher dot reduction and segment fix-up, the
    CG and LRC loops, top-k, the K7 rerank -- must give bit-identical results
    on repeated launches (any race in those protocols shows up as run-to-run
    differences)."""
    rec, n = chunglu_fixture()
    g = kz.Graph(n=n, row_offsets=rec["row_offsets"], col_indices=rec["col_indices"], original_ids=np.arange(n))
    beta = float(rec["beta"])
    idx = kz.GraphIndex(g, beta)
    op = idx.operator()
    qs = rec["queries"]
    for b, C in ((1, 1), (8, 8), (40, 8), (64, 32)):
        X = torch.randn(b * n, dtype=torch.float64, device="cuda")
        outs = []
        for _ in range(4):
            Y = torch.empty_like(X)
            d = torch.empty(b, dtype=torch.float64, device="cuda")
            op.spmm(X, Y, b=b, chunk=C, Xs=X, s1=1.0, s2=-beta, dots=d)
            outs.append((Y.clone(), d.clone()))
        for Y, d in outs[1:]:
            assert torch.equal(Y, outs[0][0]) and torch.equal(d, outs[0][1])
    runs = [kz.query_cg_baseline_batch(idx, qs, tol=1e-10, device=True) for _ in range(3)]
    for s, r in runs[1:]:
        assert torch.equal(s, runs[0][0])
        assert [x.iterations for x in r] == [x.iterations for x in runs[0][1]]
    kr = [[p.candidates for p in kz.katz_rank_batch(idx, qs, 30)] for _ in range(3)]
    assert kr[0] == kr[1] == kr[2]
    sk = [[p.candidates for p in kz.sparse_katz_batch(idx, qs[:6], 12)] for _ in range(3)]
    assert sk[0] == sk[1] == sk[2]
    li = kz.load_index(os.path.join(GOLDEN, "ba1200.klrc"))
    lq = li.id_map[::97][:12]
    lr = [kz.query_batch(li, lq, tol=1e-10) for _ in range(3)]
    for s, r in lr[1:]:
        assert np.array_equal(s, lr[0][0])
