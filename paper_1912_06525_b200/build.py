"""Offline LRC index build on the B200.

``build_index`` produces the reference's ``KatzIndex`` (index.py:104-175 of
the reference) -- and, through ``save_index``, a KLRC file the reference
can load -- for graphs whose CPU build is out of reach (the dense separator
factor of R-MAT 18 is ~27 GB).  The stages and where they run:

* partition (partition.py:178-248) and the per-part minimum-degree orders
  (factor.py:31-55): native host code in libkatzb200.so (``kz_partition``,
  ``kz_min_degree_order``), restated with the reference's tie rules, so the
  ordering is identical to the reference's;
* per-part Cholesky factors (factor.py:127-152): the parts are small
  (<= max(64, n/256) nodes); they are factored on the host with the same
  LAPACK call as the reference, batched by part size, so the factors are
  bit-identical to the reference's;
* the dense separator Cholesky M22 = L L' (factor.py:184-193) and L^-1:
  cuSOLVER/cuBLAS through torch on the device (library calls of an offline
  step, like cuBLAS for a plain GEMM);
* Lanczos with full reorthogonalisation for the top-ell eigenpairs of
  R = L^-1 M12' M11^-1 M12 L^-T (factor.py:235-319): the operator is the
  device ``KZ_LRC_CORRECTION`` apply (K1 SpMMs + the DMMA L^-1 products);
  the basis lives in HBM; the tridiagonal eigenproblem is solved on the host
  (it is at most m = max(3 ell, ell + 20) wide).  The random start vector and
  restart directions come from the same numpy Generator sequence as the
  reference's.

The built index keeps its device operands (the permuted adjacency, L^-1), so
querying it does not repeat the host-side dtrtri of a loaded index.
"""

from __future__ import annotations

import ctypes
import time
import warnings
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .factor import (BlockCholesky, DenseCholesky, FactorizationError, LazyFactors, LowRankCorrection,
                     SpectrumError)
from .graph import InadmissibleAlphaError, KatzParams, hardest_alpha, spectral_norm as _spectral_norm
from .index import BlockPartition, KatzIndex, permute_csr


class DisconnectedGraphError(ValueError):
    """Partitioning requires a connected graph (partition.py:25-26)."""


@dataclass(frozen=True)
class PartitionConfig:
    """Partitioner knobs (partition.py:29-47)."""

    max_part_size: int | None = None
    max_separator_fraction: float = 0.15
    max_recursion_depth: int = 64

    def resolved_part_size(self, n):
        if self.max_part_size is not None:
            if self.max_part_size < 1:
                raise ValueError("max_part_size must be >= 1")
            return self.max_part_size
        return max(64, n // 256)


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


def partition_vertex_separator(g, cfg=None):
    """BlockPartition of a connected graph (partition.py:178-248), computed
    by the native partitioner."""
    if g.n == 0:
        raise ValueError("empty graph")
    cfg = cfg or PartitionConfig()
    from scipy.sparse.csgraph import connected_components

    count, _ = connected_components(g.adjacency(), directed=False)
    if count != 1:
        raise DisconnectedGraphError(
            f"graph has {count} components; extract the largest component first"
        )
    limit = cfg.resolved_part_size(g.n)
    lib = _lib.load()
    rp = np.ascontiguousarray(g.row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(g.col_indices, dtype=np.int64)
    perm = np.empty(g.n, dtype=np.int64)
    bounds = np.empty(g.n + 1, dtype=np.int64)
    nparts, n1, n2 = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.check(lib.kz_partition(g.n, _ptr(rp), _ptr(ci), int(limit), int(cfg.max_recursion_depth),
                                _ptr(perm), _ptr(bounds), ctypes.byref(nparts), ctypes.byref(n1),
                                ctypes.byref(n2)))
    boundaries = bounds[: nparts.value + 1].copy()
    inv = np.empty(g.n, dtype=np.int64)
    inv[perm] = np.arange(g.n)
    overflow = n2.value > cfg.max_separator_fraction * g.n
    if overflow:
        warnings.warn(f"separator holds {n2.value}/{g.n} nodes, above the configured fraction",
                      stacklevel=2)
    return BlockPartition(perm=perm, inv_perm=inv, part_boundaries=boundaries, n1=int(n1.value),
                          n2=int(n2.value), separator_overflow=bool(overflow))


def min_degree_order(offsets, cols):
    """_min_degree_order (factor.py:31-55) of one part given its local CSR."""
    m = offsets.size - 1
    lib = _lib.load()
    rp = np.ascontiguousarray(offsets, dtype=np.int64)
    ci = np.ascontiguousarray(cols, dtype=np.int64)
    order = np.empty(m, dtype=np.int64)
    _lib.check(lib.kz_min_degree_order(m, _ptr(rp), _ptr(ci), _ptr(order)))
    return order


def _permuted_adjacency(g, bp):
    """CSR (int64 offsets, int64 cols, sorted rows) of A in partition order."""
    off, col = permute_csr(g.row_offsets, np.asarray(g.col_indices, dtype=np.int64), bp.perm, bp.inv_perm)
    rows = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(off))
    key = np.sort(rows * g.n + col.astype(np.int64))
    return off, key % g.n


def _sub_pattern(off, col, r0, r1, c0, c1):
    rows = np.repeat(np.arange(r0, r1), np.diff(off[r0 : r1 + 1]))
    cc = col[off[r0] : off[r1]]
    keep = (cc >= c0) & (cc < c1)
    rr = rows[keep] - r0
    o = np.zeros(r1 - r0 + 1, dtype=np.int64)
    np.cumsum(np.bincount(rr, minlength=r1 - r0), out=o[1:])
    return o, (cc[keep] - c0).astype(np.int64)


def block_cholesky(off, col, alpha, bounds):
    """Per-part min-degree orders and Cholesky factors of M11 = I - alpha*A11
    (factor.py:127-152); parts of equal size are factored in one batched
    LAPACK call (the same per-matrix potrf as the reference's)."""
    bounds = np.asarray(bounds, dtype=np.int64)
    nparts = bounds.size - 1
    n1 = int(bounds[-1])
    lib = _lib.load()
    rp = np.ascontiguousarray(off, dtype=np.int64)
    ci = np.ascontiguousarray(col, dtype=np.int64)
    flat = np.empty(max(n1, 1), dtype=np.int64)
    _lib.check(lib.kz_min_degree_orders(nparts, _ptr(bounds), _ptr(rp), _ptr(ci), _ptr(flat)))
    sizes = np.diff(bounds)
    part_of = np.repeat(np.arange(nparts), sizes)
    start = bounds[:-1]
    # elimination position of every interior node inside its part
    pos = np.empty(n1, dtype=np.int64)
    pos[start[part_of] + flat[:n1]] = np.arange(n1) - start[part_of]
    # interior-interior entries (both ends in the same part by construction)
    rows = np.repeat(np.arange(n1), np.diff(off[: n1 + 1]))
    cc = col[: off[n1]]
    keep = cc < n1
    rows, cc = rows[keep], cc[keep]
    orders = [flat[s : s + m].copy() for s, m in zip(start.tolist(), sizes.tolist())]
    dense = [None] * nparts
    for m in np.unique(sizes).tolist():
        members = np.flatnonzero(sizes == m)
        slot = np.empty(nparts, dtype=np.int64)
        slot[members] = np.arange(members.size)
        stack = np.zeros((members.size, m, m))
        stack[:, np.arange(m), np.arange(m)] = 1.0
        sel = sizes[part_of[rows]] == m
        r, c = rows[sel], cc[sel]
        stack[slot[part_of[r]], pos[r], pos[c]] = -alpha
        try:
            lbs = np.linalg.cholesky(stack)
        except np.linalg.LinAlgError:
            for k, p in enumerate(members.tolist()):  # name the failing part like the reference
                try:
                    np.linalg.cholesky(stack[k])
                except np.linalg.LinAlgError as err:
                    raise FactorizationError(f"part {p} is not positive definite") from err
            raise
        for k, p in enumerate(members.tolist()):
            dense[p] = lbs[k]
    factors = LazyFactors(dense)
    return BlockCholesky(block_offsets=np.asarray(bounds, dtype=np.int64), orders=orders, factors=factors,
                         dense=dense)


def _dense_m22(torch, off, col, n1, n, alpha):
    n2 = n - n1
    m22 = torch.eye(n2, dtype=torch.float64, device="cuda")
    o, c = _sub_pattern(off, col, n1, n, n1, n)
    rows = np.repeat(np.arange(n2), np.diff(o))
    if rows.size:
        r = torch.as_tensor(rows, device="cuda")
        cc = torch.as_tensor(c, device="cuda")
        m22[r, cc] = -alpha
    return m22


def dense_cholesky_device(torch, off, col, n1, n, alpha):
    """M22 = L L' (factor.py:184-193) and L^-1, on the device (peak HBM:
    three n2 x n2 doubles)."""
    m22 = _dense_m22(torch, off, col, n1, n, alpha)
    lf, info = torch.linalg.cholesky_ex(m22)
    del m22
    if int(info.item()) != 0:
        raise FactorizationError("separator block is not positive definite")
    eye = torch.eye(lf.shape[0], dtype=torch.float64, device="cuda")
    linv = torch.linalg.solve_triangular(lf, eye, upper=False)
    del eye
    return lf, linv


def _fresh_direction(torch, rng, basis):
    """_fresh_direction (factor.py:222-232) against device basis rows."""
    n = basis.shape[1]
    for _ in range(64):
        cand = torch.as_tensor(rng.standard_normal(n), device="cuda")
        for _ in range(2):
            cand -= basis.T @ (basis @ cand)
        nc = float(torch.linalg.vector_norm(cand).item())
        if nc > 1e-6:
            return cand / nc
    raise RuntimeError("could not draw a direction outside the current basis")


def lanczos_topk(apply, ell, start, max_iter=None, tol=1e-10, rng=None, psd=True, which="LA"):
    """lanczos_topk (factor.py:235-319) with the basis and the operator on
    the device; same step budget, breakdown rule, early stop and restart
    directions as the reference.  psd=False (an indefinite operator such as
    A itself) skips the reference's non-negativity check and clamp;
    which="LM" selects the ell Ritz pairs of largest magnitude instead of the
    largest algebraic values (the reference's choice)."""
    from scipy.linalg import eigh_tridiagonal

    torch = _lib.torch_cuda()
    start = np.asarray(start, dtype=np.float64)
    n = start.size
    if ell == 0 or n == 0:
        return LowRankCorrection(ell=0, vectors=np.zeros((n, 0)), values=np.zeros(0))
    if not 1 <= ell <= n:
        raise ValueError(f"rank {ell} outside [1, {n}]")
    nv = np.linalg.norm(start)
    if nv == 0.0:
        raise ValueError("start vector is zero")
    if rng is None:
        rng = np.random.default_rng(0)
    m = min(n, max(3 * ell, ell + 20)) if max_iter is None else min(n, int(max_iter))
    m = max(m, ell)
    basis = torch.zeros((m, n), dtype=torch.float64, device="cuda")  # row j = Lanczos vector j
    alphas, betas = [], []
    v = torch.as_tensor(start / nv, device="cuda")
    j = 0
    had_breakdown = False
    while True:
        basis[j] = v
        w = apply(v)
        alphas.append(float(torch.dot(v, w).item()))
        bj = basis[: j + 1]
        for _ in range(2):
            w -= bj.T @ (bj @ w)
        b = float(torch.linalg.vector_norm(w).item())
        broke = b <= 1e-8 * max(1.0, abs(alphas[-1]))
        had_breakdown = had_breakdown or broke
        j += 1
        if j >= ell:
            if j == 1:
                theta = np.asarray(alphas, dtype=np.float64)
                y = np.ones((1, 1))
            else:
                theta, y = eigh_tridiagonal(alphas, betas)
            top = np.argsort(np.abs(theta) if which == "LM" else theta)[::-1][:ell]
            resid = b * np.abs(y[-1, top])
            if (np.all(resid <= tol) and not had_breakdown) or j == m:
                break
        if broke:
            betas.append(0.0)
            v = _fresh_direction(torch, rng, basis[:j])
        else:
            betas.append(b)
            v = w / b
    vals = theta[top]
    yt = torch.as_tensor(np.ascontiguousarray(y[:, top]), device="cuda")
    vecs = (basis[:j].T @ yt).cpu().numpy()
    if psd:
        if np.any(vals < -1e-8):
            raise SpectrumError(f"negative correction eigenvalue {vals.min():.3e}")
        vals = np.maximum(vals, 0.0)
    return LowRankCorrection(ell=int(top.size), vectors=vecs, values=vals)


def build_index(g, alpha="hardest", ell=25, cfg=None, seed=0, lanczos_tol=1e-10, spectral_norm=None):
    """Build a query index for a connected graph (index.py:104-175).

    Same parameters and result as the reference's build_index;
    ``spectral_norm`` may be given to skip the device power iteration.
    """
    t0 = time.perf_counter()
    torch = _lib.torch_cuda()
    norm = float(spectral_norm) if spectral_norm is not None else _spectral_norm(g)
    if alpha == "hardest":
        alpha = hardest_alpha(norm)
    alpha = float(alpha)
    KatzParams(alpha, norm)
    if alpha < 0.0 or (alpha >= 1.0 and g.num_edges > 0):
        raise InadmissibleAlphaError(f"alpha={alpha} outside the feasible range")
    stage = {}
    t = time.perf_counter()
    bp = partition_vertex_separator(g, cfg)
    stage["partition"] = time.perf_counter() - t
    n, n1, n2 = g.n, bp.n1, bp.n2
    off, col = _permuted_adjacency(g, bp)
    # M12 = -alpha*A12 (build_blocks, partition.py:271-297)
    o12, c12 = _sub_pattern(off, col, 0, n1, n1, n)
    m12 = sp.csr_matrix((np.full(c12.size, -alpha), c12, o12), shape=(n1, n2))
    m12.sort_indices()
    t = time.perf_counter()
    bc = block_cholesky(off, col, alpha, bp.part_boundaries)
    stage["part_factors"] = time.perf_counter() - t
    ell_eff = int(min(ell, n2))
    rng = np.random.default_rng(seed)
    linv = None
    t = time.perf_counter()
    if n2 > 0:
        lf, linv = dense_cholesky_device(torch, off, col, n1, n, alpha)
        torch.cuda.synchronize()
        stage["separator_factor"] = time.perf_counter() - t
        lfac = lf.cpu().numpy()
        del lf
    else:
        lfac = np.zeros((0, 0))
    dc = DenseCholesky(factor=lfac)
    empty = LowRankCorrection(ell=0, vectors=np.zeros((n2, 0)), values=np.zeros(0))
    idx = KatzIndex(alpha=alpha, spectral_norm=norm, bp=bp, m12=m12, bc=bc, dc=dc, lr=empty,
                    id_map=g.original_ids.copy(), lanczos_seed=int(seed))
    idx.__dict__["_aperm"] = (off, col)
    if linv is not None:
        # the padded row-major L^-1 and L^-T operands DeviceLRC uploads for a
        # loaded index, made here without leaving the device
        ld = n2 + (n2 & 1)
        cache = idx._op_cache()
        pad = torch.zeros((n2, ld), dtype=torch.float64, device="cuda")
        pad[:, :n2] = linv.tril_()
        cache["linv_pad"] = pad
        pad = torch.zeros((n2, ld), dtype=torch.float64, device="cuda")
        pad[:, :n2] = linv.T
        cache["linvT_pad"] = pad
        del linv
    t = time.perf_counter()
    if ell_eff > 0:
        start = rng.standard_normal(n2)
        dev = idx.lrc()  # ell = 0 operands: enough for the correction apply
        lr = lanczos_topk(dev.apply_correction_device, ell_eff, start, tol=lanczos_tol, rng=rng)
        idx._op_cache().pop("lrc", None)
        del dev
    else:
        lr = empty
    idx.lr = lr
    stage["lanczos"] = time.perf_counter() - t
    nnz11 = int(off[n1] - np.count_nonzero(col[: off[n1]] >= n1))  # off-diagonal entries of A11
    m11_nnz = nnz11 + n1
    idx.build_stats = {
        "n": g.n,
        "num_edges": g.num_edges,
        "alpha": alpha,
        "spectral_norm": norm,
        "n1": n1,
        "n2": n2,
        "num_parts": bp.num_parts,
        "separator_fraction": n2 / g.n if g.n else 0.0,
        "separator_overflow": bp.separator_overflow,
        "m11_nnz": m11_nnz,
        "interior_factor_nnz": bc.nnz,
        "fill_ratio": bc.nnz / max(1, (m11_nnz + n1) // 2),
        "correction_rank": lr.ell,
        "correction_values": [float(s) for s in lr.values],
        "build_seconds": time.perf_counter() - t0,
        "stage_seconds": stage,
    }
    return idx
