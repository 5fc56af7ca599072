"""Device operands of the LRC-Katz solve and the Python entry points.

``DeviceLRC(idx)`` re-expresses a loaded KLRC index once for the GPU:

* A in partition order, split into the K1 operators A12 (n1 x n2),
  A21 (n2 x n1) and A22 (n2 x n2); M12 = -alpha*A12 exactly (the index
  stores M12 with every value -alpha, index.py:52-67);
* M11^-1 as a weighted block-diagonal K1 operator: per part b the dense
  inverse (Lb Lb')^-1 mapped back through the part's order, i.e. the
  operator BlockCholesky.solve applies (factor.py:89-106) without the
  per-part Python loop;
* L^-1 (LAPACK dtrtri, once) and its transpose, row-major, so each
  preconditioner application is two triangular products instead of four
  triangular solves (factor.py:331-337);
* U row-major and (U diag(d))^T with d = 1/(1-sigma) - 1 (factor.py:336).

The handle borrows these tensors; they live as long as this object.
"""

from __future__ import annotations

import ctypes

import numpy as np
from scipy.linalg import lapack

from . import _lib
from .graph import DeviceOperator


def _sub_csr(off, col, r0, r1, c0, c1):
    """Rows [r0, r1) x cols [c0, c1) of a CSR (column indices shifted by c0)."""
    rows = np.repeat(np.arange(r0, r1), np.diff(off[r0 : r1 + 1]))
    cc = col[off[r0] : off[r1]]
    keep = (cc >= c0) & (cc < c1)
    rr = rows[keep] - r0
    offsets = np.zeros(r1 - r0 + 1, dtype=np.int64)
    np.cumsum(np.bincount(rr, minlength=r1 - r0), out=offsets[1:])
    return offsets, (cc[keep] - c0).astype(np.int32)


def interior_inverse_csr(idx):
    """CSR (rows n1) of M11^-1 from the per-part Cholesky factors."""
    bo = idx.bc.block_offsets
    n1 = idx.n1
    sizes = np.diff(bo)
    offsets = np.zeros(n1 + 1, dtype=np.int64)
    np.cumsum(np.repeat(sizes, sizes), out=offsets[1:])
    nnz = int(offsets[-1])
    cols = np.empty(nnz, dtype=np.int32)
    vals = np.empty(nnz, dtype=np.float64)
    # parts of equal size are inverted together (R-MAT 18 has ~10^5 parts,
    # most of size 1): W = Lb^-T Lb^-1 = (Lb Lb')^-1 in elimination order,
    # scattered back through the part's order o: row o[i], column o[j]
    for m in np.unique(sizes).tolist():
        if m == 0:
            continue
        members = np.flatnonzero(sizes == m)
        lbs = np.stack([idx.bc.dense[b] for b in members.tolist()])
        if m == 1:
            w = 1.0 / (lbs * lbs)
        else:
            li = np.tril(np.linalg.inv(lbs))
            w = np.matmul(np.transpose(li, (0, 2, 1)), li)
        os_ = np.stack([np.asarray(idx.bc.orders[b], dtype=np.int64) for b in members.tolist()])
        wl = np.empty_like(w)
        k = np.arange(members.size)[:, None, None]
        wl[k, os_[:, :, None], os_[:, None, :]] = w
        starts = bo[members]
        p0 = offsets[starts]
        span = (p0[:, None] + np.arange(m * m)[None, :]).ravel()
        cols[span] = (starts[:, None, None] + np.zeros((1, m, 1), np.int64) + np.arange(m)[None, None, :]).reshape(-1)
        vals[span] = wl.reshape(-1)
    return offsets, cols, vals


def pad_even(torch, a):
    """Row-major device copy with the leading dimension rounded up to even,
    zero padded (the kernels load entry pairs as one 16-byte access)."""
    a = np.asarray(a, dtype=np.float64)
    rows, cols = a.shape
    out = np.zeros((rows, cols + (cols & 1)))
    out[:, :cols] = a
    return torch.as_tensor(out).cuda()


class DeviceLRC:
    """kz_lrc handle plus the device tensors it borrows."""

    def __init__(self, idx):
        torch = _lib.torch_cuda()
        lib = _lib.load()
        self.lib = lib
        self.idx = idx
        n, n1, n2, ell = idx.n, idx.n1, idx.n2, int(idx.lr.ell)
        self.n, self.n1, self.n2, self.ell = n, n1, n2, ell
        off, col = idx.adjacency_permuted()
        self.full = idx.operator()
        self.a12 = self.a21 = self.a22 = self.minv = None
        if n1 > 0 and n2 > 0:
            o, c = _sub_csr(off, col, 0, n1, n1, n)
            self.a12 = DeviceOperator(o, c, n1, n2)
            o, c = _sub_csr(off, col, n1, n, 0, n1)
            self.a21 = DeviceOperator(o, c, n2, n1)
        if n2 > 0:
            o, c = _sub_csr(off, col, n1, n, n1, n)
            self.a22 = DeviceOperator(o, c, n2, n2)
        if n1 > 0:
            o, c, v = interior_inverse_csr(idx)
            h = ctypes.c_void_p()
            _lib.check(lib.kz_graph_create_weighted(n1, n1, int(o[-1]), o.ctypes.data, c.ctypes.data,
                                                    v.ctypes.data, ctypes.byref(h)))
            self.minv = _Handle(lib, h)
        def dev(a):
            return pad_even(torch, a)

        self.t_linv = self.t_linvT = self.t_u = self.t_udT = None
        sigma = np.ascontiguousarray(idx.lr.values[:ell], dtype=np.float64)
        if n2 > 0:
            cache = idx._op_cache()
            if "linv_pad" in cache:  # device-built index (build.py): L^-1 never left HBM
                self.t_linv, self.t_linvT = cache["linv_pad"], cache["linvT_pad"]
            else:
                lf = np.asarray(idx.dc.factor, dtype=np.float64)
                linv, info = lapack.dtrtri(lf, lower=1)
                if info != 0:
                    raise RuntimeError("separator factor is singular")
                linv = np.tril(linv)
                self.t_linv = dev(linv)
                self.t_linvT = dev(linv.T)
            if ell > 0:
                u = np.asarray(idx.lr.vectors, dtype=np.float64)[:, :ell]
                with np.errstate(divide="ignore"):
                    d = 1.0 / (1.0 - sigma) - 1.0
                self.t_u = dev(u)
                self.t_udT = dev((u * d).T)
        desc = _lib.KzLrcDesc()
        desc.n, desc.n1, desc.n2, desc.ell = n, n1, n2, ell
        desc.beta = float(idx.alpha)
        desc.full = self.full.handle.value
        desc.a12 = self.a12.handle.value if self.a12 else None
        desc.a21 = self.a21.handle.value if self.a21 else None
        desc.a22 = self.a22.handle.value if self.a22 else None
        desc.minv = self.minv.handle.value if self.minv else None
        desc.linv = self.t_linv.data_ptr() if self.t_linv is not None else None
        desc.linvT = self.t_linvT.data_ptr() if self.t_linvT is not None else None
        desc.u = self.t_u.data_ptr() if self.t_u is not None else None
        desc.udT = self.t_udT.data_ptr() if self.t_udT is not None else None
        self._sigma = sigma
        desc.sigma = ctypes.cast(sigma.ctypes.data, ctypes.POINTER(ctypes.c_double)) if ell > 0 else None
        h = ctypes.c_void_p()
        _lib.check(lib.kz_lrc_create(ctypes.byref(desc), ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.kz_lrc_destroy(h)
            except Exception:
                pass
            self.handle = None

    # -- batched query / pcg ------------------------------------------------
    def _run(self, b, qpos=None, f=None, tol=1e-8, max_iter=None, start_seed=None, perm=None,
             clamp=True, out_rows=None):
        torch = _lib.torch_cuda()
        lib = self.lib
        out = torch.empty((b, out_rows), dtype=torch.float64, device="cuda")
        x0 = None
        if start_seed is not None and self.n2 > 0:
            from .solver import _start_vector

            x0 = torch.as_tensor(_start_vector(self.n2, start_seed), dtype=torch.float64).cuda()
        reps = (_lib.KzReport * b)()
        ms = ctypes.c_float(0.0)
        args = _lib.KzLrcArgs()
        args.b = b
        args.chunk = 0
        args.clamp = 1 if clamp else 0
        keep = []
        if qpos is not None:
            arr, p = _lib.i64_array(qpos)
            keep.append(arr)
            args.qpos = p
        args.f = f.data_ptr() if f is not None else None
        args.tol = float(tol)
        args.max_iter = int(max_iter) if max_iter is not None else 0
        args.x0 = x0.data_ptr() if x0 is not None else None
        args.perm = perm.data_ptr() if perm is not None else None
        args.out = out.data_ptr()
        args.reports = ctypes.cast(reps, ctypes.POINTER(_lib.KzReport))
        args.device_ms = ctypes.pointer(ms)
        nbytes = lib.kz_lrc_workspace_bytes(self.handle, b, 0)
        ws = _lib.Workspace.get(torch, nbytes, slot="lrc")
        _lib.check(lib.kz_lrc_batch(self.handle, ctypes.byref(args), _lib.ptr(ws), ws.numel(),
                                    _lib.stream_ptr(torch)))
        return out, reps, ms.value

    def query_batch(self, positions, tol=1e-8, max_iter=None, start_seed=None):
        from .solver import _batches

        torch = _lib.torch_cuda()
        positions = np.asarray(positions, dtype=np.int64)
        b = positions.size
        scores = torch.empty((b, self.n), dtype=torch.float64, device="cuda")
        reports, total_ms = [], 0.0
        perm = self.idx.device_perm()
        for s, e in _batches(b, 4 * self.n + 8 * max(self.n2, 1)):
            out, reps, ms = self._run(e - s, qpos=positions[s:e], tol=tol, max_iter=max_iter,
                                      start_seed=start_seed, perm=perm, out_rows=self.n)
            scores[s:e] = out
            reports.extend(reps)
            total_ms += ms
        return scores, reports, total_ms

    def pcg(self, f, tol=1e-8, max_iter=None, start_seed=None):
        """lrc_pcg (solver.py:118-158) on one Schur right-hand side."""
        from .solver import SolveReport

        torch = _lib.torch_cuda()
        as_numpy = isinstance(f, np.ndarray) or not hasattr(f, "is_cuda")
        ft = torch.as_tensor(np.asarray(f, dtype=np.float64) if as_numpy else f,
                             dtype=torch.float64).cuda().reshape(1, -1).contiguous()
        if ft.shape[1] != self.n2:
            raise ValueError("right-hand side has the wrong length")
        if self.n2 == 0:  # solver.py:127-152 with an empty system: x = [], converged at 0 iterations
            x = torch.zeros(0, dtype=torch.float64, device="cuda")
            rep = SolveReport(iterations=0, final_residual_norm=0.0, converged=True, wall_time=0.0)
            return (x.cpu().numpy() if as_numpy else x), rep
        out, reps, ms = self._run(1, f=ft, tol=tol, max_iter=max_iter, start_seed=start_seed,
                                  clamp=False, out_rows=self.n2)
        r = reps[0]
        rep = SolveReport(iterations=int(r.iterations), final_residual_norm=float(r.final_residual_norm),
                          converged=bool(r.converged), wall_time=ms / 1e3)
        x = out[0]
        return (x.cpu().numpy() if as_numpy else x), rep

    # -- single operator applications (kz_lrc_apply) --------------------------
    def _apply(self, op, in1, in2, rows_out):
        torch = _lib.torch_cuda()
        lib = self.lib
        a = torch.as_tensor(np.asarray(in1, dtype=np.float64)).cuda().reshape(1, -1).contiguous()
        b2 = None
        if in2 is not None:
            b2 = torch.as_tensor(np.asarray(in2, dtype=np.float64)).cuda().reshape(1, -1).contiguous()
        out = torch.empty((1, rows_out), dtype=torch.float64, device="cuda")
        ws = _lib.Workspace.get(torch, lib.kz_lrc_workspace_bytes(self.handle, 1, 1), slot="lrc_apply")
        _lib.check(lib.kz_lrc_apply(self.handle, op, 1, _lib.ptr(a), _lib.ptr(b2), _lib.ptr(out),
                                    _lib.ptr(ws), ws.numel(), _lib.stream_ptr(torch)))
        return out[0].cpu().numpy()

    def apply_correction_device(self, v):
        """R v (factor.py:196-202) for a device vector of length n2."""
        torch = _lib.torch_cuda()
        lib = self.lib
        a = v.reshape(1, -1).contiguous()
        out = torch.empty((1, self.n2), dtype=torch.float64, device="cuda")
        ws = _lib.Workspace.get(torch, lib.kz_lrc_workspace_bytes(self.handle, 1, 1), slot="lrc_apply")
        _lib.check(lib.kz_lrc_apply(self.handle, 3, 1, _lib.ptr(a), None, _lib.ptr(out),
                                    _lib.ptr(ws), ws.numel(), _lib.stream_ptr(torch)))
        return out[0]

    def apply_correction(self, v):
        return self._apply(3, v, None, self.n2)

    def apply_schur(self, v):
        if self.n2 == 0:
            if np.size(v) != 0:
                raise ValueError("vector has the wrong length")
            return np.zeros(0)
        return self._apply(0, v, None, self.n2)

    def apply_precond(self, r):
        return self._apply(1, r, None, self.n2)

    def schur_rhs(self, g1, g2):
        return self._apply(2, g1, g2, self.n2)


class _Handle:
    def __init__(self, lib, h):
        self.lib, self.handle = lib, h

    def __del__(self):
        if self.handle is not None and self.handle.value:
            try:
                self.lib.kz_graph_destroy(self.handle)
            except Exception:
                pass
            self.handle = None


def lrc_query_batch(idx, positions, tol=1e-8, max_iter=None, start_seed=None):
    """query() for many partition positions: returns (scores cuda [b][n] in
    internal order, [SolveReport])."""
    from .solver import SolveReport

    scores, reps, ms = idx.lrc().query_batch(positions, tol=tol, max_iter=max_iter, start_seed=start_seed)
    reports = [SolveReport(iterations=int(r.iterations), final_residual_norm=float(r.final_residual_norm),
                           converged=bool(r.converged), wall_time=ms / 1e3) for r in reps]
    return scores, reports


def device_gram(lf):
    """L L^T on the device (index load helper for the separator adjacency)."""
    torch = _lib.torch_cuda()
    t = torch.as_tensor(np.ascontiguousarray(lf, dtype=np.float64)).cuda()
    return (t @ t.T).cpu().numpy()
