"""The reference's partition/factor helpers under their own names and
signatures (partition.py:250-297, factor.py:127-202, 322-337), for callers
that use them directly.  The query hot path does not go through these (it
runs on the operands lrc.py uploads once); they exist so a user of lrckatz
finds every public name.  Device work is done with torch on the GPU (cuBLAS /
cuSOLVER / cuSPARSE for these offline helpers) and the native partitioner /
min-degree code of libkatzb200.so.

* build_blocks(g, alpha, bp) -> (M11, M12, M22) scipy CSR, M = I - alpha*A in
  partition order (partition.py:271-297);
* check_partition(g, bp) -> bool (partition.py:250-268);
* block_cholesky(m11, block_offsets) -> BlockCholesky (factor.py:127-152):
  min-degree orders (native) and per-part LAPACK potrf batched by part size,
  the same factors as the reference;
* dense_cholesky(m22) -> DenseCholesky (factor.py:184-193), cuSOLVER;
* apply_correction(dc, m12, bc, v) = L^-1 M12' M11^-1 M12 L^-T v
  (factor.py:196-202) and apply_approx_schur_inverse(dc, lr, r)
  (factor.py:322-337), on the device.
"""

from __future__ import annotations

import ctypes

import numpy as np
import scipy.sparse as sp

from . import _lib
from .factor import BlockCholesky, DenseCholesky, FactorizationError, LazyFactors, SpectrumError
from .graph import InadmissibleAlphaError


def build_blocks(g, alpha, bp):
    """(M11, M12, M22) of M = I - alpha*A under the partition order."""
    from .build import _permuted_adjacency

    if alpha < 0.0 or (alpha >= 1.0 and g.num_edges > 0):
        raise InadmissibleAlphaError(f"alpha={alpha} outside the feasible range")
    off, col = _permuted_adjacency(g, bp)
    n, n1 = g.n, bp.n1
    a = sp.csr_matrix((np.full(col.size, -float(alpha)), col, off), shape=(n, n))
    m = (sp.identity(n, format="csr") + a).tocsr()
    m.eliminate_zeros()  # alpha == 0 leaves explicit zeros
    m11, m12, m22 = m[:n1, :n1].tocsr(), m[:n1, n1:].tocsr(), m[n1:, n1:].tocsr()
    for blk in (m11, m12, m22):
        blk.sort_indices()
    return m11, m12, m22


def check_partition(g, bp):
    """True iff bp is a valid interior/separator ordering of g."""
    n = g.n
    if bp.n1 + bp.n2 != n or np.shape(bp.perm) != (n,) or np.shape(bp.inv_perm) != (n,):
        return False
    if not np.array_equal(np.sort(bp.perm), np.arange(n)):
        return False
    if not np.array_equal(bp.perm[bp.inv_perm], np.arange(n)):
        return False
    b = np.asarray(bp.part_boundaries)
    if b[0] != 0 or b[-1] != bp.n1 or np.any(np.diff(b) < 0):
        return False
    part_of = np.full(n, -1, dtype=np.int64)  # -1: separator
    sizes = np.diff(b)
    part_of[bp.perm[: bp.n1]] = np.repeat(np.arange(sizes.size), sizes)
    rows = np.repeat(np.arange(n), np.diff(g.row_offsets))
    pu, pw = part_of[rows], part_of[g.col_indices]
    return not np.any((pu >= 0) & (pw >= 0) & (pu != pw))


def block_cholesky(m11, block_offsets):
    """Per-part min-degree orders and Cholesky factors of a block-diagonal
    M11 (any values); FactorizationError names the failing part."""
    m11 = sp.csr_matrix(m11)
    bounds = np.asarray(block_offsets, dtype=np.int64)
    nparts = bounds.size - 1
    n1 = int(bounds[-1])
    lib = _lib.load()
    rp = np.ascontiguousarray(m11.indptr, dtype=np.int64)
    ci = np.ascontiguousarray(m11.indices, dtype=np.int64)
    flat = np.empty(max(n1, 1), dtype=np.int64)
    _lib.check(lib.kz_min_degree_orders(nparts, ctypes.c_void_p(bounds.ctypes.data), ctypes.c_void_p(rp.ctypes.data),
                                        ctypes.c_void_p(ci.ctypes.data), ctypes.c_void_p(flat.ctypes.data)))
    sizes = np.diff(bounds)
    part_of = np.repeat(np.arange(nparts), sizes)
    start = bounds[:-1]
    pos = np.empty(n1, dtype=np.int64)
    pos[start[part_of] + flat[:n1]] = np.arange(n1) - start[part_of]
    coo = m11.tocoo()
    rows, cols, vals = coo.row.astype(np.int64), coo.col.astype(np.int64), coo.data
    orders = [flat[s : s + m].copy() for s, m in zip(start.tolist(), sizes.tolist())]
    dense = [None] * nparts
    for m in np.unique(sizes).tolist():
        if m == 0:
            continue
        members = np.flatnonzero(sizes == m)
        slot = np.empty(nparts, dtype=np.int64)
        slot[members] = np.arange(members.size)
        stack = np.zeros((members.size, m, m))
        sel = sizes[part_of[rows]] == m
        stack[slot[part_of[rows[sel]]], pos[rows[sel]], pos[cols[sel]]] = vals[sel]
        try:
            lbs = np.linalg.cholesky(stack)
        except np.linalg.LinAlgError:
            for k, p in enumerate(members.tolist()):
                try:
                    np.linalg.cholesky(stack[k])
                except np.linalg.LinAlgError as err:
                    raise FactorizationError(f"part {p} is not positive definite") from err
            raise
        for k, p in enumerate(members.tolist()):
            dense[p] = lbs[k]
    for p in np.flatnonzero(sizes == 0).tolist():
        dense[p] = np.zeros((0, 0))
    return BlockCholesky(block_offsets=bounds, orders=orders, factors=LazyFactors(dense), dense=dense)


def dense_cholesky(m22):
    """M22 = L L' on the device (cuSOLVER)."""
    a = m22.toarray() if sp.issparse(m22) else np.asarray(m22, dtype=np.float64)
    if a.size == 0:
        return DenseCholesky(factor=np.zeros((a.shape[0], a.shape[0])))
    torch = _lib.torch_cuda()
    lf, info = torch.linalg.cholesky_ex(torch.as_tensor(a, dtype=torch.float64, device="cuda"))
    if int(info.item()) != 0:
        raise FactorizationError("separator block is not positive definite")
    return DenseCholesky(factor=lf.cpu().numpy())


# -- device applications ------------------------------------------------------
_cache = {}


def _dev(torch, key, make):
    """Device copy of a host operand, cached per (tag, object identity)."""
    tag, obj = key
    k = (tag, id(obj))
    hit = _cache.get(k)
    if hit is None or hit[0] is not obj:
        hit = (obj, make())
        _cache[k] = hit
    return hit[1]


def _dev_factor(torch, dc):
    return _dev(torch, ("L", dc), lambda: torch.as_tensor(np.asarray(dc.factor), dtype=torch.float64, device="cuda"))


def _solve_lower(torch, lf, v, transpose=False):
    if transpose:  # L^-T v
        return torch.linalg.solve_triangular(lf.T, v.reshape(-1, 1), upper=True).reshape(-1)
    return torch.linalg.solve_triangular(lf, v.reshape(-1, 1), upper=False).reshape(-1)


def apply_correction(dc, m12, bc, v):
    """R v = L^-1 M12' M11^-1 M12 L^-T v (factor.py:196-202) on the device."""
    from .lrc import interior_inverse_csr

    torch = _lib.torch_cuda()
    lf = _dev_factor(torch, dc)
    key12 = m12  # cache on the caller's object
    m12 = sp.csr_matrix(m12)
    n1 = m12.shape[0]
    vt = torch.as_tensor(np.asarray(v, dtype=np.float64), device="cuda")
    y = _solve_lower(torch, lf, vt, transpose=True)
    if n1 == 0:
        return np.zeros(np.shape(v))
    s12 = _dev(torch, ("M12", key12), lambda: torch.sparse_csr_tensor(
        torch.as_tensor(m12.indptr, dtype=torch.int64), torch.as_tensor(m12.indices, dtype=torch.int64),
        torch.as_tensor(m12.data, dtype=torch.float64), size=m12.shape).cuda())
    s21 = _dev(torch, ("M21", key12), lambda: (lambda t: torch.sparse_csr_tensor(
        torch.as_tensor(t.indptr, dtype=torch.int64), torch.as_tensor(t.indices, dtype=torch.int64),
        torch.as_tensor(t.data, dtype=torch.float64), size=t.shape).cuda())(m12.T.tocsr()))

    class _Shim:  # interior_inverse_csr reads .bc and .n1
        pass

    def make_minv():
        sh = _Shim()
        sh.bc, sh.n1 = bc, n1
        o, c, w = interior_inverse_csr(sh)
        return torch.sparse_csr_tensor(torch.as_tensor(o, dtype=torch.int64), torch.as_tensor(c, dtype=torch.int64),
                                       torch.as_tensor(w, dtype=torch.float64), size=(n1, n1)).cuda()

    minv = _dev(torch, ("Minv", bc), make_minv)
    w1 = s12 @ y
    u = minv @ w1
    z = s21 @ u
    return _solve_lower(torch, lf, z).cpu().numpy()


def apply_approx_schur_inverse(dc, lr, r):
    """L^-T (I + U D U') L^-1 r, D = 1/(1 - sigma) - 1 (factor.py:322-337)."""
    vals = np.asarray(lr.values, dtype=np.float64)
    if np.any(vals >= 1.0):
        raise SpectrumError("correction eigenvalue at or above 1")
    torch = _lib.torch_cuda()
    lf = _dev_factor(torch, dc)
    rt = torch.as_tensor(np.asarray(r, dtype=np.float64), device="cuda")
    t = _solve_lower(torch, lf, rt)
    if lr.ell:
        u = _dev(torch, ("U", lr), lambda: torch.as_tensor(np.asarray(lr.vectors), dtype=torch.float64, device="cuda"))
        d = torch.as_tensor(1.0 / (1.0 - vals) - 1.0, device="cuda")
        t = t + u @ ((u.T @ t) * d)
    return _solve_lower(torch, lf, t, transpose=True).cpu().numpy()
