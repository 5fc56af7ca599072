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
import threading

import numpy as np
import scipy.sparse as sp
from scipy.linalg import lapack

from . import _lib
from .factor import BlockCholesky, DenseCholesky, FactorizationError, LazyFactors, SpectrumError
from .graph import DeviceOperator, InadmissibleAlphaError


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
# apply_correction / apply_approx_schur_inverse run on the library's own
# kernels (kz_lrc_apply: K1 SpMMs and the DMMA L^-1 products), through a
# kz_lrc handle built from exactly the operands the reference function
# receives and cached per operand identity.
_cache = {}
_lock = threading.Lock()


def _cached(key, objs, make):
    """make() once per (key, identity of objs); the cached value keeps the
    objects alive so their ids stay unique."""
    k = (key,) + tuple(id(o) for o in objs)
    with _lock:
        hit = _cache.get(k)
        if hit is None or any(a is not b for a, b in zip(hit[0], objs)):
            hit = (tuple(objs), make())
            _cache[k] = hit
        return hit[1]


class _FactorHandle:
    """A kz_lrc handle over (L, U, sigma) and optionally M12 / M11^-1: the
    operands of apply_approx_schur_inverse (factor.py:322-337) or
    apply_correction (factor.py:196-202).  M12 is a weighted K1 operator with
    the caller's values (beta = -1 so the kernels' -beta*M12 x is M12 x)."""

    def __init__(self, dc, lr=None, m12=None, bc=None):
        from .lrc import _Handle, interior_inverse_csr, pad_even

        torch = _lib.torch_cuda()
        lib = _lib.load()
        self.lib = lib
        lf = np.asarray(dc.factor, dtype=np.float64)
        n2 = lf.shape[0]
        n1 = 0 if m12 is None else int(m12.shape[0])
        ell = 0 if lr is None else int(lr.ell)
        self.n1, self.n2, self.ell = n1, n2, ell
        n = n1 + n2
        empty = np.zeros(n + 1, dtype=np.int64)
        self.full = DeviceOperator(empty, np.zeros(0, dtype=np.int32), n)
        self.a22 = DeviceOperator(np.zeros(n2 + 1, dtype=np.int64), np.zeros(0, dtype=np.int32), n2)
        self.a12 = self.a21 = self.minv = None
        if n1 > 0:
            m = sp.csr_matrix(m12)
            m.sort_indices()
            mt = m.T.tocsr()
            mt.sort_indices()

            def weighted(c, rows, cols):
                h = ctypes.c_void_p()
                o = np.ascontiguousarray(c.indptr, dtype=np.int64)
                ci = np.ascontiguousarray(c.indices, dtype=np.int32)
                v = np.ascontiguousarray(c.data, dtype=np.float64)
                _lib.check(lib.kz_graph_create_weighted(rows, cols, int(o[-1]), o.ctypes.data, ci.ctypes.data,
                                                        v.ctypes.data, ctypes.byref(h)))
                return _Handle(lib, h)

            self.a12 = weighted(m, n1, n2)
            self.a21 = weighted(mt, n2, n1)

            class _Parts:  # interior_inverse_csr reads .bc and .n1
                pass

            sh = _Parts()
            sh.bc, sh.n1 = bc, n1
            o, c, w = interior_inverse_csr(sh)
            self.minv = weighted(sp.csr_matrix((w, c, o), shape=(n1, n1)), n1, n1)
        linv, info = lapack.dtrtri(lf, lower=1)
        if info != 0:
            raise FactorizationError("separator factor is singular")
        linv = np.tril(linv)
        self.t_linv = pad_even(torch, linv)
        self.t_linvT = pad_even(torch, linv.T)
        self.t_u = self.t_udT = None
        sigma = np.zeros(0)
        if ell > 0:
            sigma = np.ascontiguousarray(lr.values[:ell], dtype=np.float64)
            u = np.asarray(lr.vectors, dtype=np.float64)[:, :ell]
            with np.errstate(divide="ignore"):
                d = 1.0 / (1.0 - sigma) - 1.0
            self.t_u = pad_even(torch, u)
            self.t_udT = pad_even(torch, (u * d).T)
        self._sigma = sigma
        desc = _lib.KzLrcDesc()
        desc.n, desc.n1, desc.n2, desc.ell = n, n1, n2, ell
        desc.beta = -1.0
        desc.full = self.full.handle.value
        desc.a12 = self.a12.handle.value if self.a12 else None
        desc.a21 = self.a21.handle.value if self.a21 else None
        desc.a22 = self.a22.handle.value
        desc.minv = self.minv.handle.value if self.minv else None
        desc.linv, desc.linvT = self.t_linv.data_ptr(), self.t_linvT.data_ptr()
        desc.u = self.t_u.data_ptr() if self.t_u is not None else None
        desc.udT = self.t_udT.data_ptr() if self.t_udT is not None else None
        desc.sigma = ctypes.cast(sigma.ctypes.data, ctypes.POINTER(ctypes.c_double)) if ell > 0 else None
        h = ctypes.c_void_p()
        _lib.check(lib.kz_lrc_create(ctypes.byref(desc), ctypes.byref(h)))
        self.handle = h

    def apply(self, op, v):
        torch = _lib.torch_cuda()
        lib = self.lib
        x = torch.as_tensor(np.asarray(v, dtype=np.float64)).cuda().reshape(1, -1).contiguous()
        out = torch.empty((1, self.n2), dtype=torch.float64, device="cuda")
        ws = _lib.Workspace.get(torch, lib.kz_lrc_workspace_bytes(self.handle, 1, 1), slot="lrc_apply")
        _lib.check(lib.kz_lrc_apply(self.handle, op, 1, _lib.ptr(x), None, _lib.ptr(out), _lib.ptr(ws), ws.numel(),
                                    _lib.stream_ptr(torch)))
        return out[0].cpu().numpy()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.kz_lrc_destroy(h)
            except Exception:
                pass
            self.handle = None


_KZ_LRC_PRECOND = 1
_KZ_LRC_CORRECTION = 3


def apply_correction(dc, m12, bc, v):
    """R v = L^-1 M12' M11^-1 M12 L^-T v (factor.py:196-202) on the device:
    kz_lrc_apply(KZ_LRC_CORRECTION) -- K1 SpMMs with M12 / M11^-1 and the
    DMMA L^-1 products."""
    n2 = np.asarray(dc.factor).shape[0]
    if np.shape(v) != (n2,):
        raise ValueError("vector has the wrong length")
    if n2 == 0 or sp.csr_matrix(m12).shape[0] == 0:
        return np.zeros(n2)
    h = _cached("corr", (dc, m12, bc), lambda: _FactorHandle(dc, m12=m12, bc=bc))
    return h.apply(_KZ_LRC_CORRECTION, v)


def apply_approx_schur_inverse(dc, lr, r):
    """L^-T (I + U D U') L^-1 r, D = 1/(1 - sigma) - 1 (factor.py:322-337), on
    the device: kz_lrc_apply(KZ_LRC_PRECOND) (DMMA L^-1 products, the
    low-rank term on the same kernels)."""
    vals = np.asarray(lr.values, dtype=np.float64)
    if np.any(vals >= 1.0):
        raise SpectrumError("correction eigenvalue at or above 1")
    n2 = np.asarray(dc.factor).shape[0]
    if np.shape(r) != (n2,):
        raise ValueError("vector has the wrong length")
    if n2 == 0:
        return np.zeros(0)
    h = _cached("precond", (dc, lr), lambda: _FactorHandle(dc, lr=lr))
    return h.apply(_KZ_LRC_PRECOND, r)
