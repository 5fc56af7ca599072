"""CPU oracle for the Katz query hot path -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference's query path
(/root/reference/pkg/src/lrckatz, cited file:line below), used as the
checker by tests/, by __graft_entry__.smoke() and by bench.py's
cpu_baseline / --impl reference legs.  The product package
(paper_1912_06525_b200) never imports this module.

Pinning: the restatement is checked against golden vectors produced by the
reference itself (tests/golden/make_golden.py imports /root/reference in the
build container) -- see tests/test_oracle_golden.py.  The arithmetic
boundary is numpy/scipy exactly as in the reference (pyproject.toml:10-13
pins numpy>=1.24, scipy>=1.10; no lock file).
"""

from __future__ import annotations

import hashlib
import struct
import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
from scipy.linalg import solve_triangular


@dataclass(frozen=True)
class Report:
    iterations: int
    final_residual_norm: float
    converged: bool
    wall_time: float


# ---------------------------------------------------------------------------
# solver.py:51-101 -- textbook CG
# ---------------------------------------------------------------------------


def initial_state(b, start_seed, apply_a):
    """solver.py:51-59"""
    if start_seed is None:
        return np.zeros(b.size), b.copy()
    x = np.random.default_rng(start_seed).standard_normal(b.size)
    nx = np.linalg.norm(x)
    if nx > 0:
        x /= nx
    return x, b - apply_a(x)


def cg(apply_a, b, tol=1e-8, max_iter=None, start_seed=None, x0=None):
    """solver.py:62-101; x0 (not in the reference) replaces the seeded start
    of _initial_state (solver.py:51-59) by a given vector."""
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    if max_iter is None:
        max_iter = 10 * n
    t0 = time.perf_counter()
    thresh = tol * np.linalg.norm(b)
    if x0 is not None:
        x = np.array(x0, dtype=np.float64)
        r = b - apply_a(x)
    else:
        x, r = initial_state(b, start_seed, apply_a)
    rnorm = np.linalg.norm(r)
    it = 0
    if rnorm > thresh:
        p = r.copy()
        rs = float(r @ r)
        while it < max_iter:
            q = apply_a(p)
            pq = float(p @ q)
            if pq <= 0.0:
                raise RuntimeError("operator is not positive definite")
            a = rs / pq
            x += a * p
            r -= a * q
            it += 1
            rs_new = float(r @ r)
            rnorm = np.sqrt(rs_new)
            if rnorm <= thresh:
                break
            p = r + (rs_new / rs) * p
            rs = rs_new
    return x, Report(it, float(rnorm), bool(rnorm <= thresh), time.perf_counter() - t0)


# ---------------------------------------------------------------------------
# CSR restatement of query_cg_baseline: the reference's own
# cg recurrence with apply_a = v - beta*(A@v) on a scipy CSR, rhs beta*A e_q,
# clamp at 0 (solver.py:210-232)
# ---------------------------------------------------------------------------


def csr_matrix(row_offsets, col_indices, n):
    return sp.csr_matrix((np.ones(len(col_indices)), np.asarray(col_indices), np.asarray(row_offsets)),
                         shape=(n, n))


def query_cg_csr(a, beta, q, tol=1e-8, max_iter=None, start_seed=None):
    """Scores (clamped) and report of one query on CSR adjacency a."""
    n = a.shape[0]
    rhs = np.zeros(n)
    rhs[a.indices[a.indptr[q] : a.indptr[q + 1]]] = beta
    x, rep = cg(lambda v: v - beta * (a @ v), rhs, tol, max_iter, start_seed)
    return np.maximum(x, 0.0), rep


# ---------------------------------------------------------------------------
# Eigen-form LRC (the north star's "low-rank term from a
# top-r eigen index of A plus a CG correction", not in the reference): the
# start is the Galerkin point x0 = U W U'b of the index basis (U'b = beta
# (AU)[q,:] for b = beta A e_q), then the reference's cg recurrence from x0
# with r0 = b - M x0 formed by the operator (the device forms it from AU;
# the two agree to roundoff).  U, AU (n x r, internal order) and W come from
# the device index (EigenIndex.basis_internal).
# ---------------------------------------------------------------------------


def query_eigen_csr(a, beta, q, u, au, w, tol=1e-8, max_iter=None, a2u=None, a3u=None, a4u=None):
    """Scores (clamped) and report of one query, eigen-form start + cg.
    With a2u (= A^2 U) the walk start: x0 = beta A e_q + U y with
    y = beta^2 W (A^2 U)[q]' (the Galerkin step on the remainder)."""
    n = a.shape[0]
    rhs = np.zeros(n)
    rhs[a.indices[a.indptr[q] : a.indptr[q + 1]]] = beta
    if a4u is not None:
        # three-term walk start: x0 = beta A e_q + beta^2 A^2 e_q + beta^3 A^3 e_q + U y,
        # y = beta^4 W (A^4 U)[q]'
        y = (beta ** 4) * (w @ a4u[q])
        a2e = a @ (a @ np.eye(1, n, q).ravel())
        x0 = rhs + (beta * beta) * a2e + (beta ** 3) * (a @ a2e) + u @ y
    elif a3u is not None:
        # two-term walk start: x0 = beta A e_q + beta^2 A^2 e_q + U y,
        # y = beta^3 W (A^3 U)[q]'
        y = (beta * beta * beta) * (w @ a3u[q])
        x0 = rhs + (beta * beta) * (a @ (a @ np.eye(1, n, q).ravel())) + u @ y
    elif a2u is None:
        y = beta * (w @ au[q])
        x0 = u @ y
    else:
        y = (beta * beta) * (w @ a2u[q])
        x0 = rhs + u @ y
    x, rep = cg(lambda v: v - beta * (a @ v), rhs, tol, max_iter, x0=x0)
    return np.maximum(x, 0.0), rep


# ---------------------------------------------------------------------------
# KLRC reader (index.py:228-333) and the factor arithmetic (factor.py)
# ---------------------------------------------------------------------------


@dataclass(eq=False)
class OracleIndex:
    alpha: float
    spectral_norm: float
    n: int
    n1: int
    n2: int
    ell: int
    id_map: np.ndarray
    perm: np.ndarray
    inv_perm: np.ndarray
    bounds: np.ndarray
    m12: sp.csr_matrix
    orders: list
    dense: list
    L: np.ndarray
    U: np.ndarray
    sigma: np.ndarray

    def internal_id(self, original):
        pos = int(np.searchsorted(self.id_map, original))
        if pos == self.n or self.id_map[pos] != original:
            raise KeyError(f"unknown node id {original}")
        return pos


def read_klrc(path_or_bytes):
    """Plain KLRC reader (no validation beyond the checksum)."""
    data = path_or_bytes if isinstance(path_or_bytes, bytes) else open(path_or_bytes, "rb").read()
    assert data[:4] == b"KLRC"
    assert hashlib.blake2b(data[:-8], digest_size=8).digest() == data[-8:]
    pos = 25
    alpha, norm = struct.unpack_from("<dd", data, 9)
    _, n, n1, n2, ell, nparts = struct.unpack_from("<6Q", data, pos)
    pos += 48

    def ints(c):
        nonlocal pos
        out = np.frombuffer(data, "<i8", c, pos).astype(np.int64)
        pos += 8 * c
        return out

    def flts(c):
        nonlocal pos
        out = np.frombuffer(data, "<f8", c, pos).astype(np.float64)
        pos += 8 * c
        return out

    def csr(r, c):
        nonlocal pos
        (nnz,) = struct.unpack_from("<Q", data, pos)
        pos += 8
        ip, ix, dv = ints(r + 1), ints(nnz), flts(nnz)
        return sp.csr_matrix((dv, ix, ip), shape=(r, c))

    id_map, perm, bounds = ints(n), ints(n), ints(nparts + 1)
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    m12 = csr(n1, n2)
    orders, dense = [], []
    for b in range(nparts):
        size = int(bounds[b + 1] - bounds[b])
        orders.append(ints(size))
        dense.append(csr(size, size).toarray())
    L = np.asfortranarray(flts(n2 * n2).reshape((n2, n2), order="F"))
    U = np.asfortranarray(flts(n2 * ell).reshape((n2, ell), order="F"))
    sigma = flts(ell)
    return OracleIndex(alpha, norm, int(n), int(n1), int(n2), int(ell), id_map, perm, inv, bounds,
                       m12, orders, dense, L, U, sigma)


def bc_solve(ix, x):
    """BlockCholesky.solve (factor.py:89-106)"""
    out = np.empty_like(x)
    for b in range(len(ix.dense)):
        s, e = int(ix.bounds[b]), int(ix.bounds[b + 1])
        o, lb = ix.orders[b], ix.dense[b]
        z = x[s:e][o]
        y = solve_triangular(lb, z, lower=True, check_finite=False)
        y = solve_triangular(lb, y, lower=True, trans=1, check_finite=False)
        buf = np.empty(e - s)
        buf[o] = y
        out[s:e] = buf
    return out


def bc_multiply(ix, x):
    """BlockCholesky.multiply (factor.py:108-124)"""
    out = np.empty_like(x)
    for b in range(len(ix.dense)):
        s, e = int(ix.bounds[b]), int(ix.bounds[b + 1])
        o, lb = ix.orders[b], ix.dense[b]
        y = lb @ (lb.T @ x[s:e][o])
        buf = np.empty(e - s)
        buf[o] = y
        out[s:e] = buf
    return out


def dc_solve(ix, r):
    """DenseCholesky.solve (factor.py:170-172)"""
    y = solve_triangular(ix.L, r, lower=True, check_finite=False)
    return solve_triangular(ix.L, y, lower=True, trans=1, check_finite=False)


def dc_multiply(ix, v):
    """DenseCholesky.multiply (factor.py:180-181)"""
    return ix.L @ (ix.L.T @ v)


def apply_m_permuted(ix, x):
    """KatzIndex.apply_m_permuted (index.py:86-91)"""
    x1, x2 = x[: ix.n1], x[ix.n1 :]
    top = bc_multiply(ix, x1) + ix.m12 @ x2
    bottom = ix.m12.T @ x1 + dc_multiply(ix, x2)
    return np.concatenate([top, bottom])


def rhs_for_position(ix, pos):
    """index.py:93-101"""
    e = np.zeros(ix.n)
    e[pos] = 1.0
    return e - apply_m_permuted(ix, e)


def schur_rhs(ix, g1, g2):
    """solver.py:104-110"""
    if ix.n2 == 0:
        return np.zeros(0)
    return g2 - ix.m12.T @ bc_solve(ix, g1)


def apply_schur(ix, v):
    """solver.py:113-115"""
    return dc_multiply(ix, v) - ix.m12.T @ bc_solve(ix, ix.m12 @ v)


def apply_approx_schur_inverse(ix, r):
    """factor.py:322-337"""
    if np.any(ix.sigma >= 1.0):
        raise RuntimeError("correction eigenvalue at or above 1")
    base = dc_solve(ix, r)
    if ix.ell == 0:
        return base
    t = solve_triangular(ix.L, r, lower=True, check_finite=False)
    c = ix.U.T @ t
    c *= 1.0 / (1.0 - ix.sigma) - 1.0
    return base + solve_triangular(ix.L, ix.U @ c, lower=True, trans=1, check_finite=False)


def lrc_pcg(ix, f, tol=1e-8, max_iter=None, start_seed=None):
    """solver.py:118-158"""
    f = np.asarray(f, dtype=np.float64)
    n = f.size
    if max_iter is None:
        max_iter = 10 * n
    t0 = time.perf_counter()
    thresh = tol * np.linalg.norm(f)
    x, r = initial_state(f, start_seed, lambda v: apply_schur(ix, v))
    rnorm = np.linalg.norm(r)
    it = 0
    if rnorm > thresh:
        z = apply_approx_schur_inverse(ix, r)
        p = z.copy()
        rz = float(r @ z)
        while it < max_iter:
            q = apply_schur(ix, p)
            pq = float(p @ q)
            if pq <= 0.0:
                raise RuntimeError("Schur operator is not positive definite")
            a = rz / pq
            x += a * p
            r -= a * q
            it += 1
            rnorm = float(np.linalg.norm(r))
            if rnorm <= thresh:
                break
            z = apply_approx_schur_inverse(ix, r)
            rz_new = float(r @ z)
            p = z + (rz_new / rz) * p
            rz = rz_new
    return x, Report(it, float(rnorm), bool(rnorm <= thresh), time.perf_counter() - t0)


def query_lrc(ix, q, tol=1e-8, max_iter=None, start_seed=None):
    """query / _solve_query_system (solver.py:161-207); q is an original id."""
    pos = ix.inv_perm[ix.internal_id(q)]
    t0 = time.perf_counter()
    rhs = rhs_for_position(ix, pos)
    rhs_norm = np.linalg.norm(rhs)
    g1, g2 = rhs[: ix.n1], rhs[ix.n1 :]
    if ix.n2 == 0:
        k1 = bc_solve(ix, g1)
        k2 = np.zeros(0)
        inner = Report(0, 0.0, True, 0.0)
    else:
        f = schur_rhs(ix, g1, g2)
        fnorm = np.linalg.norm(f)
        tol_eff = tol * rhs_norm / fnorm if fnorm > 0 else tol
        k2, inner = lrc_pcg(ix, f, tol_eff, max_iter, start_seed)
        k1 = bc_solve(ix, g1 - ix.m12 @ k2)
    k_perm = np.concatenate([k1, k2])
    resid = float(np.linalg.norm(rhs - apply_m_permuted(ix, k_perm)))
    scores = np.empty(ix.n)
    scores[ix.perm] = k_perm
    np.maximum(scores, 0.0, out=scores)
    return scores, Report(inner.iterations, resid, bool(resid <= tol * rhs_norm),
                          time.perf_counter() - t0)


def query_cg_index(ix, q, tol=1e-8, max_iter=None, start_seed=None):
    """query_cg_baseline (solver.py:210-232) on a KLRC index."""
    pos = ix.inv_perm[ix.internal_id(q)]
    rhs = rhs_for_position(ix, pos)
    k_perm, inner = cg(lambda v: apply_m_permuted(ix, v), rhs, tol, max_iter, start_seed)
    scores = np.empty(ix.n)
    scores[ix.perm] = k_perm
    np.maximum(scores, 0.0, out=scores)
    return scores, inner


def index_adjacency_internal(ix):
    """A in internal order from the factors (test helper)."""
    n = ix.n
    m = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        m[:, j] = e - apply_m_permuted(ix, e)
    a_perm = (m > ix.alpha / 2).astype(np.float64)
    a = np.zeros_like(a_perm)
    a[np.ix_(ix.perm, ix.perm)] = a_perm
    return sp.csr_matrix(a)


# ---------------------------------------------------------------------------
# linkpred.py:115-207 -- scoring, with a pluggable solver
# ---------------------------------------------------------------------------


def pearson(x, y):
    """linkpred.py:115-133"""
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


def candidate_order(n, scores, internal, neighbors, s):
    """linkpred.py:145-152"""
    mask = np.ones(n, dtype=bool)
    mask[internal] = False
    mask[neighbors] = False
    cand = np.flatnonzero(mask)
    order = np.lexsort((cand, -scores[cand]))
    return cand[order[: s if s is not None else cand.size]]


def katz_rank(solve, neighbors_of, id_map, q_internal, s):
    """linkpred.py:155-162; solve(internal) -> scores, neighbors_of(internal)."""
    scores = solve(q_internal)
    n = scores.size
    top = candidate_order(n, scores, q_internal, neighbors_of(q_internal), s)
    return [(int(id_map[x]), float(scores[x])) for x in top]


def sparse_katz(solve, neighbors_of, id_map, q_internal, s, T=None):
    """linkpred.py:165-207"""
    if T is None:
        T = s + 1
    scores = solve(q_internal)
    n = scores.size
    top = candidate_order(n, scores, q_internal, neighbors_of(q_internal), s)
    if top.size == 0:
        return []
    order = np.lexsort((np.arange(n), -scores))
    anchors = [x for x in order if x != q_internal][:T]
    ref = np.empty(T + 1)
    ref[0] = scores[q_internal]
    ref[1:] = scores[anchors]
    profiles = np.empty((T + 1, top.size))
    profiles[0] = scores[top]
    for i, t_int in enumerate(anchors):
        profiles[1 + i] = solve(int(t_int))[top]
    ref_c = ref - ref.mean()
    sr = np.linalg.norm(ref_c)
    pc = profiles - profiles.mean(axis=0)
    sp_ = np.linalg.norm(pc, axis=0)
    corr = np.zeros(top.size)
    ok = (sp_ > 0.0) & (sr > 0.0)
    if sr > 0.0:
        corr[ok] = np.clip((ref_c @ pc[:, ok]) / (sr * sp_[ok]), -1.0, 1.0)
    rerank = np.lexsort((top, -scores[top], -corr))
    return [(int(id_map[top[i]]), float(corr[i])) for i in rerank]


# ---------------------------------------------------------------------------
# Input preparation for bench.py --impl reference and the scale tests: the
# seeded generators of SURVEY.md Appendix B, from_edges (graph.py:111-148),
# the largest component (graph.py:232-261) and spectral_norm (graph.py:264-297)
# restated on numpy/scipy only, so the reference arm loads nothing from the
# product package.  tests/test_oracle_golden.py checks them against the
# reference's own from_edges / largest_connected_component / spectral_norm
# outputs (tests/golden/ingest.npz, chunglu2000_cg.npz).
# ---------------------------------------------------------------------------

RMAT_ABCD = (0.57, 0.19, 0.19, 0.05)


def rmat_pairs(scale, edge_factor=16, abcd=RMAT_ABCD, seed=0):
    """SURVEY Appendix B R-MAT: one uniform per edge and bit, least
    significant bit first; u_bit = r >= a+b, v_bit = (a <= r < a+b) or
    r >= a+b+c."""
    a, b, c, _ = abcd
    n = 1 << scale
    m = n * edge_factor
    rng = np.random.default_rng(seed)
    u = np.zeros(m, dtype=np.int64)
    v = np.zeros(m, dtype=np.int64)
    for bit in range(scale):
        r = rng.random(m)
        u |= (r >= a + b).astype(np.int64) << bit
        v |= (((r >= a) & (r < a + b)) | (r >= a + b + c)).astype(np.int64) << bit
        del r
    return u, v, n


def chung_lu_pairs(n=10_000, gamma=2.5, mean_degree=10.0, seed=0):
    """SURVEY Appendix B Chung-Lu: weights i^(-1/(gamma-1)) scaled to the
    mean degree, n*d/2 pairs drawn i.i.d. proportional to them (u batch
    first, then v)."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-1.0 / (gamma - 1.0))
    w *= mean_degree / w.mean()
    p = w / w.sum()
    m = int(n * mean_degree / 2)
    rng = np.random.default_rng(seed)
    u = rng.choice(n, size=m, p=p)
    v = rng.choice(n, size=m, p=p)
    return u, v, n


def from_pairs(u, v, n):
    """graph.py:111-148 from_edges: drop self-loops, symmetrise, deduplicate,
    columns sorted within each row.  Returns (row_offsets, col_indices)."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    keep = u != v
    u, v = u[keep], v[keep]
    a = sp.coo_matrix((np.ones(u.size, dtype=np.int8), (u, v)), shape=(n, n)).tocsr()
    a = (a + a.T).tocsr()
    a.sum_duplicates()
    a.sort_indices()
    return a.indptr.astype(np.int64), a.indices.astype(np.int64)


def largest_component(row_offsets, col_indices, n, original_ids=None):
    """graph.py:232-261: the largest connected component, ties to the one
    holding the smallest id (the reference labels components in order of
    their smallest node), relabelled contiguously in increasing id order.
    Returns (row_offsets, col_indices, original_ids)."""
    from scipy.sparse.csgraph import connected_components

    if original_ids is None:
        original_ids = np.arange(n, dtype=np.int64)
    a = sp.csr_matrix((np.ones(len(col_indices), dtype=np.int8), col_indices, row_offsets), shape=(n, n))
    count, labels = connected_components(a, directed=False)
    if count == 1:
        return np.asarray(row_offsets), np.asarray(col_indices), np.asarray(original_ids)
    sizes = np.bincount(labels, minlength=count)
    first = np.full(count, n, dtype=np.int64)
    np.minimum.at(first, labels, np.arange(n))
    big = np.flatnonzero(sizes == sizes.max())
    best = big[np.argmin(first[big])]
    keep = np.flatnonzero(labels == best)
    sub = a[keep][:, keep].tocsr()
    sub.sort_indices()
    return sub.indptr.astype(np.int64), sub.indices.astype(np.int64), np.asarray(original_ids)[keep].copy()


def spectral_norm(a, tol=1e-7, max_iter=10000):
    """graph.py:264-297: power iteration on A @ A from the uniform positive
    vector; returns ||A v|| of the final unit iterate."""
    n = a.shape[0]
    if a.nnz == 0:
        return 0.0
    v = np.full(n, 1.0 / np.sqrt(n))
    last = 0.0
    for _ in range(max_iter):
        w = a @ (a @ v)
        est = np.sqrt(v @ w)
        nw = np.linalg.norm(w)
        if nw == 0.0:
            return 0.0
        v = w / nw
        if abs(est - last) <= tol * max(est, 1e-300):
            return float(np.linalg.norm(a @ v))
        last = est
    raise RuntimeError(f"spectral norm estimate did not settle in {max_iter} iterations")


def config_csr(cfg, seed=0):
    """(row_offsets, col_indices, original_ids) of a BASELINE config graph
    after the largest component: cfg1 Chung-Lu 10^4, cfg2 R-MAT 18,
    cfg3 R-MAT 22, proxy16 R-MAT 16."""
    if cfg == "cfg1":
        u, v, n = chung_lu_pairs(seed=seed)
    else:
        u, v, n = rmat_pairs({"proxy16": 16, "cfg2": 18, "cfg3": 22}[cfg], seed=seed)
    off, col = from_pairs(u, v, n)
    del u, v
    return largest_component(off, col, n)


def sample_queries(id_map, count, seed=0):
    """cli.py:119-120: sort(default_rng(seed).choice(id_map, count, replace=False))."""
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(np.asarray(id_map), size=count, replace=False))


# BASELINE.json per-config query batch, top-k and tolerance (the bench's
# reference arm reads them here; tests check they equal generators.CONFIGS)
BENCH_CONFIGS = {
    "cfg1": dict(b=16, k=20, tol=1e-8),
    "proxy16": dict(b=64, k=50, tol=1e-8),
    "cfg2": dict(b=64, k=50, tol=1e-8),
    "cfg3": dict(b=256, k=100, tol=1e-8),
}
