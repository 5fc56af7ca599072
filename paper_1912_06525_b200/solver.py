"""Katz query solvers on the GPU, with the reference's Python API.

Mirrors lrckatz.solver (solver.py:1-232): ``cg``, ``lrc_pcg``,
``schur_rhs``, ``apply_schur``, ``query``, ``query_cg_baseline`` and the
``SolveReport`` / ``KatzVector`` types, plus batched entry points
(``query_batch``, ``query_cg_baseline_batch``) that solve many query
columns in one device call.  All arithmetic runs in libkatzb200.so
(K1 SpMM, K2 CG, the LRC kernels); this module only marshals arguments.

Semantics kept from the reference:
  * a query solves (I - alpha*A) k = alpha*A e_q and returns scores in
    internal node order, clamped at zero (solver.py:181-184, 223-225);
  * per-column stop rule ||r|| <= tol*||rhs||, default max_iter 10*n;
  * ``UnknownNodeError`` (a KeyError) for ids outside the index;
  * ``RuntimeError`` when p.q <= 0; non-convergence is reported, not raised.
``wall_time`` of a batched call is the batch's device time (CUDA events),
shared by every column of the batch.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib


class UnknownNodeError(KeyError):
    """Query node id is not in the indexed graph (solver.py:25-26)."""


@dataclass(frozen=True)
class SolveReport:
    iterations: int
    final_residual_norm: float
    converged: bool
    wall_time: float


@dataclass(eq=False)
class KatzVector:
    """Katz proximities of every node to the query (solver.py:37-48)."""

    scores: np.ndarray
    query: int
    alpha: float


def _start_vector(n, start_seed):
    """The seeded start of _initial_state (solver.py:51-59)."""
    x = np.random.default_rng(start_seed).standard_normal(n)
    nx = np.linalg.norm(x)
    if nx > 0:
        x /= nx
    return x


def _positions(idx, qs):
    try:
        internal = idx.internal_ids(qs)
    except KeyError as err:
        raise UnknownNodeError(str(err)) from None
    return internal, idx.solve_positions(internal)


# largest block (in doubles) one device call may allocate per solve vector,
# and the most query columns one call takes
_MAX_BLOCK_DOUBLES = 2_000_000_000
_MAX_COLUMNS = 8192


def _batches(b, n):
    per = max(1, min(b, _MAX_COLUMNS, _MAX_BLOCK_DOUBLES // max(n, 1)))
    for s in range(0, b, per):
        yield s, min(b, s + per)


def cg_solve_device(idx, positions, tol=1e-8, max_iter=None, start_seed=None, rhs=None,
                    out=None, clamp=True, perm=True, eigen=False):
    """Batched CG on the index operator.  Returns (scores[b][n] cuda fp64,
    kz reports, device ms).  Scores are scattered to internal order when the
    index is permuted (perm=True).  eigen=True (an EigenIndex, query columns,
    no seeded start) starts every column at the eigen-of-A Galerkin point
    (kz_eigen_batch)."""
    torch = _lib.torch_cuda()
    lib = _lib.load()
    op = idx.operator()
    n = idx.n
    positions = np.asarray(positions, dtype=np.int64)
    b = int(positions.size) if rhs is None else int(rhs.shape[0])
    if out is None:
        out = torch.empty((b, n), dtype=torch.float64, device="cuda")
    x0 = None
    if start_seed is not None:
        xs = _start_vector(n, start_seed)
        # the seeded vector lives in the reference's solve space: partition
        # order for a KLRC index, internal order for a GraphIndex
        if hasattr(idx, "start_vector_to_solve"):
            xs = idx.start_vector_to_solve(xs)
        x0 = torch.as_tensor(xs, dtype=torch.float64).cuda()
    dperm = idx.device_perm() if perm else None
    reports = (_lib.KzReport * b)()
    total_ms = 0.0
    st = _lib.stream_ptr(torch)
    for s, e in _batches(b, n):
        nb = e - s
        qarr, qptr = _lib.i64_array(positions[s:e] if rhs is None else np.zeros(nb))
        ms = ctypes.c_float(0.0)
        args = _lib.KzCgArgs()
        args.b = nb
        args.clamp = 1 if clamp else 0
        args.qpos = qptr if rhs is None else ctypes.POINTER(ctypes.c_int64)()
        args.rhs = rhs[s:e].data_ptr() if rhs is not None else None
        args.beta = float(idx.alpha)
        args.tol = float(tol)
        args.max_iter = int(max_iter) if max_iter is not None else 0
        args.x0 = x0.data_ptr() if x0 is not None else None
        args.perm = dperm.data_ptr() if dperm is not None else None
        args.scores = out[s:e].data_ptr()
        sub = (_lib.KzReport * nb).from_address(ctypes.addressof(reports) + s * ctypes.sizeof(_lib.KzReport))
        args.reports = ctypes.cast(sub, ctypes.POINTER(_lib.KzReport))
        args.device_ms = ctypes.pointer(ms)
        if eigen:
            eh = idx.eigen_handle()
            wsb = lib.kz_eigen_workspace_bytes(eh, nb)
            ws = _lib.Workspace.get(torch, wsb, slot="cg")
            rc = lib.kz_eigen_batch(eh, ctypes.byref(args), _lib.ptr(ws), ws.numel(), st)
        else:
            wsb = lib.kz_cg_workspace_bytes(op.handle, nb)
            ws = _lib.Workspace.get(torch, wsb, slot="cg")
            rc = lib.kz_cg_batch(op.handle, ctypes.byref(args), _lib.ptr(ws), ws.numel(), st)
        _lib.check(rc)
        total_ms += ms.value
    return out, reports, total_ms


def _reports(kz_reports, wall, use_true=None):
    out = []
    for j, r in enumerate(kz_reports):
        out.append(SolveReport(iterations=int(r.iterations),
                               final_residual_norm=float(r.final_residual_norm),
                               converged=bool(r.converged), wall_time=wall))
    return out


def query_cg_baseline_batch(idx, qs, tol=1e-8, max_iter=None, start_seed=None, device=False):
    """query_cg_baseline for many queries in one device call.

    Returns (scores, reports): scores is a cuda fp64 tensor [b][n] (internal
    order) when device=True, else a numpy array.  The report of each column
    carries its own iteration count and CG's recursive residual
    (solver.py:226-231)."""
    qs = np.atleast_1d(np.asarray(qs, dtype=np.int64))
    _, pos = _positions(idx, qs)
    scores, reps, ms = cg_solve_device(idx, pos, tol=tol, max_iter=max_iter, start_seed=start_seed)
    reports = _reports(reps, ms / 1e3)
    if device:
        return scores, reports
    return scores.cpu().numpy(), reports


def query_cg_baseline(idx, q, tol=1e-8, max_iter=None, start_seed=None):
    """Plain CG on the full (permuted) system (solver.py:210-232)."""
    scores, reports = query_cg_baseline_batch(idx, [q], tol, max_iter, start_seed)
    return KatzVector(scores=scores[0], query=int(q), alpha=idx.alpha), reports[0]


def query_batch(idx, qs, tol=1e-8, max_iter=None, start_seed=None, device=False):
    """query() for many queries in one device call.

    KatzIndex: LRC-Katz Schur PCG (solver.py:194-207).  EigenIndex: the
    eigen-of-A low-rank start + CG correction (north-star LRC; a seeded
    start falls back to plain CG from that start).  GraphIndex (no factors):
    plain CG, the only solver such an index supports."""
    qs = np.atleast_1d(np.asarray(qs, dtype=np.int64))
    kind = getattr(idx, "solver_kind", "cg")
    if kind == "eigen" and start_seed is None:
        _, pos = _positions(idx, qs)
        scores, reps, ms = cg_solve_device(idx, pos, tol=tol, max_iter=max_iter, eigen=True)
        reports = _reports(reps, ms / 1e3)
        return (scores, reports) if device else (scores.cpu().numpy(), reports)
    if kind != "lrc":
        return query_cg_baseline_batch(idx, qs, tol, max_iter, start_seed, device)
    from .lrc import lrc_query_batch

    _, pos = _positions(idx, qs)
    scores, reports = lrc_query_batch(idx, pos, tol=tol, max_iter=max_iter, start_seed=start_seed)
    if device:
        return scores, reports
    return scores.cpu().numpy(), reports


def query(idx, q, tol=1e-8, max_iter=None, start_seed=None):
    """Exact Katz proximity vector for original id q (solver.py:194-207)."""
    scores, reports = query_batch(idx, [q], tol, max_iter, start_seed)
    return KatzVector(scores=scores[0], query=int(q), alpha=idx.alpha), reports[0]


# ---------------------------------------------------------------------------
# generic CG on a caller-supplied operator (solver.py:62-101)
# ---------------------------------------------------------------------------


class KatzOperator:
    """v -> v - beta*A v on the device: the operator cg() runs fully in one
    kz_cg_batch call (pass it as apply_a)."""

    def __init__(self, op, beta):
        self.op = op
        self.beta = float(beta)

    def __call__(self, v):
        torch = _lib.torch_cuda()
        x = torch.as_tensor(v, dtype=torch.float64).cuda().contiguous()
        y = torch.empty_like(x)
        self.op.spmm(x, y, b=1, Xs=x, s1=1.0, s2=-self.beta)
        return y if not isinstance(v, np.ndarray) else y.cpu().numpy()


class _OpIndex:
    def __init__(self, op, alpha, n):
        self._op, self.alpha, self.n = op, alpha, n

    def operator(self):
        return self._op

    def device_perm(self):
        return None


def cg(apply_a, b, tol=1e-8, max_iter=None, start_seed=None):
    """Plain conjugate gradient (solver.py:62-101); returns (x, SolveReport).

    With a KatzOperator the whole solve is one kz_cg_batch call.  Any other
    callable is applied to CUDA tensors each iteration while the vector
    arithmetic (dots via kz_coldot) stays on the device."""
    as_numpy = isinstance(b, np.ndarray) or not hasattr(b, "is_cuda")
    torch = _lib.torch_cuda()
    bt = torch.as_tensor(np.asarray(b, dtype=np.float64) if as_numpy else b,
                         dtype=torch.float64).cuda().contiguous().reshape(-1)
    n = bt.numel()
    if isinstance(apply_a, KatzOperator):
        scores, reps, ms = cg_solve_device(_OpIndex(apply_a.op, apply_a.beta, n), np.zeros(1),
                                           tol=tol, max_iter=max_iter, start_seed=start_seed,
                                           rhs=bt.reshape(1, n), clamp=False, perm=False)
        x = scores[0]
        rep = _reports(reps, ms / 1e3)[0]
        return (x.cpu().numpy() if as_numpy else x), rep
    return _generic_cg(apply_a, bt, tol, max_iter, start_seed, as_numpy, torch)


def _dot(torch, x, y):
    lib = _lib.load()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.coldot(torch, lib, x, y, out, x.numel())
    return float(out.item())


def _axpby(torch, a, x, b, y, out):
    """out = a*x + b*y on the device (kz_vec_op; numpy's rounding)."""
    _lib.vec_op(torch, _lib.load(), 0, x.numel(), a, x, b, y, out)


def _generic_cg(apply_a, bt, tol, max_iter, start_seed, as_numpy, torch):
    n = bt.numel()
    if max_iter is None:
        max_iter = 10 * n
    t0 = time.perf_counter()

    def apply(v):
        y = apply_a(v.cpu().numpy() if as_numpy else v)
        return torch.as_tensor(np.asarray(y, dtype=np.float64) if as_numpy else y,
                               dtype=torch.float64).cuda().reshape(-1)

    thresh = tol * np.sqrt(_dot(torch, bt, bt))
    if start_seed is None:
        x = torch.zeros_like(bt)
        r = torch.empty_like(bt)
        _axpby(torch, 1.0, bt, 0.0, None, r)  # r = b
    else:
        x = torch.as_tensor(_start_vector(n, start_seed), dtype=torch.float64).cuda()
        r = bt - apply(x)
    rnorm = np.sqrt(_dot(torch, r, r))
    it = 0
    if rnorm > thresh:
        p = torch.empty_like(r)
        _axpby(torch, 1.0, r, 0.0, None, p)  # p = r
        rs = _dot(torch, r, r)
        while it < max_iter:
            q = apply(p)
            pq = _dot(torch, p, q)
            if pq <= 0.0:
                raise RuntimeError("operator is not positive definite")
            a = rs / pq
            _axpby(torch, a, p, 1.0, x, x)  # x += a*p
            _axpby(torch, -a, q, 1.0, r, r)  # r -= a*q
            it += 1
            rs_new = _dot(torch, r, r)
            rnorm = np.sqrt(rs_new)
            if rnorm <= thresh:
                break
            _axpby(torch, rs_new / rs, p, 1.0, r, p)  # p = r + (rs_new/rs)*p
            rs = rs_new
    rep = SolveReport(iterations=it, final_residual_norm=float(rnorm),
                      converged=bool(rnorm <= thresh), wall_time=time.perf_counter() - t0)
    return (x.cpu().numpy() if as_numpy else x), rep


def _apply_m_host(idx, x):
    """M x = x - alpha*A x in partition order, computed by K1 (index.py:86-91)."""
    return KatzOperator(idx.operator(), idx.alpha)(np.asarray(x, dtype=np.float64))


def schur_rhs(idx, g1, g2):
    """f = g2 - M12' M11^-1 g1 (solver.py:104-110), on the device."""
    if np.shape(g1) != (idx.n1,) or np.shape(g2) != (idx.n2,):
        raise ValueError("right-hand side blocks have wrong lengths")
    if idx.n2 == 0:
        return np.zeros(0)
    return idx.lrc().schur_rhs(g1, g2)


def apply_schur(idx, v):
    """S v = M22 v - M12' M11^-1 M12 v (solver.py:113-115), on the device."""
    return idx.lrc().apply_schur(v)


def lrc_pcg(idx, f, tol=1e-8, max_iter=None, start_seed=None):
    """Schur-complement PCG with the low-rank corrected preconditioner
    (solver.py:118-158), on the device.  Returns (x, SolveReport)."""
    return idx.lrc().pcg(f, tol=tol, max_iter=max_iter, start_seed=start_seed)
