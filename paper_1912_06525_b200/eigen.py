"""Eigen-of-A low-rank index: the north-star form of LRC-Katz.

BASELINE.json's north star describes LRC-Katz as "a low-rank term from a
precomputed index of top-r eigenpairs (U, Lambda) of the symmetric adjacency
A, plus a Conjugate Gradient correction on (I - beta A) x = residual".  The
reference's own LRC is the Schur-complement form (lrc.py / kz_lrc_*); this
is the other one, not in the reference, so its parity is
against the exact solution (tests/test_gpu_eigen.py).

``EigenIndex(graph_index, rank)`` wraps a ``GraphIndex`` (same operator, same
solve order, same ids) and adds, in that order:

* U: the ``rank`` Ritz vectors of A of largest |eigenvalue| (``which="LM"``,
  default; "LA" = largest algebraic) by the device Lanczos of build.py (K1
  SpMMs with b = 1, full reorthogonalisation, basis in HBM).  Both ends of
  the spectrum bound CG's rate on I - beta A: deflating the most negative
  eigenvalues as well cuts R-MAT 22 from 7 to 5 CG iterations per batch
  (largest algebraic alone: 6);
* AU = A U: one K1 SpMM of the r-column block;
* T = U'AU and W = (I - beta T)^-1 (r x r).

* A^(m+1) U for the m-term walk start (``walk_terms`` m = 1, 2, 3; 3 is the
  default): m more K1 SpMMs of the r-column block.

A query's low-rank term is the Galerkin point of span(U),
x0 = U W U' b with U' b = beta (AU)[q, :]' -- exact for any orthonormal U, so
Ritz-vector accuracy only changes iteration counts -- and the CG correction
runs from x0 with the exact residual r0 = b - x0 + beta (AU) W U' b; both
products are the two tall-skinny fp64 DMMA GEMMs of ``lowrank_init_kernel``
(one fused pass), then the reference's CG recurrence (solver.py:62-101) with
the stop test ||r|| <= tol ||b||.

Walk start (``walk_terms=1``): the first Katz-series term beta A e_q goes
into the start exactly and the Galerkin step is taken on the remainder,
x0 = beta A e_q + U y with y = beta^2 W (A^2 U)[q, :]', so
r0 = beta^2 A^2 e_q - U y + beta (AU) y, where A^2 e_q is the integer count
of 2-walks from q (a sparse push over the neighbours' lists, order-free
integer atomics).  Measured effect: the CG correction needs one iteration
fewer (R-MAT 16 prototype: 5 -> 4 at r = 128, 5.5 -> 4.5 at r = 32).

Two-term walk start (``walk_terms=2``): x0 = beta A e_q + beta^2 A^2 e_q + U y
with y = beta^3 W (A^3 U)[q, :]' (the Galerkin step on the remainder
beta^3 A^3 e_q); the 2-walk counts give the second term, and r0 = b - M x0
comes from one K1 SpMM on x0 -- which replaces the (AU) y GEMM of the start --
so one more CG iteration disappears for the price of that SpMM.

Three-term walk start (``walk_terms=3``, the default above 10^6 stored
entries; one term below): x0 also carries
beta^3 A^3 e_q, one K1 SpMM on the beta^2 A^2 e_q block, and y uses A^4 U;
R-MAT 22: 2 CG iterations instead of 3 (1.97 mean).
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _lib
from .index import GraphIndex


class EigenIndex:
    """GraphIndex + top-r eigen basis of A (solver_kind "eigen")."""

    solver_kind = "eigen"

    def __init__(self, gi, rank, lanczos_tol=1e-8, seed=0, max_steps=None, which="LM", walk_terms=None):
        from .build import lanczos_topk

        if not isinstance(gi, GraphIndex):
            raise TypeError("EigenIndex wraps a GraphIndex")
        torch = _lib.torch_cuda()
        lib = _lib.load()
        self.gi = gi
        self.alpha = gi.alpha
        self.spectral_norm = gi.spectral_norm
        self.id_map = gi.id_map
        n = gi.n
        rank = int(rank)
        if not 1 <= rank <= min(n, 384):
            raise ValueError(f"rank {rank} outside [1, min(n, 384)]")
        if walk_terms is None:
            # each extra term costs one SpMM in the start and removes one CG
            # iteration (SpMM + vector passes): a win once SpMMs dominate the
            # launch overheads -- measured: cfg1 (10^5 entries) is fastest with
            # one term, R-MAT 16-22 (10^6-10^8) with three
            walk_terms = 3 if gi.graph.nnz > 1_000_000 else 1
        if walk_terms not in (0, 1, 2, 3):
            raise ValueError("walk_terms must be 0 (Galerkin start), 1, 2 or 3 (Katz terms put in exactly)")
        self.walk_terms = int(walk_terms)
        t0 = time.perf_counter()
        op = gi.operator()

        def apply(v):
            y = torch.empty_like(v)
            op.spmm(v, y, b=1)
            return y

        rng = np.random.default_rng(seed)
        lr = lanczos_topk(apply, rank, rng.standard_normal(n), max_iter=max_steps, tol=lanczos_tol, rng=rng,
                          psd=False, which=which)
        t_lanczos = time.perf_counter() - t0
        r = int(lr.ell)
        ldr = (r + 3) // 4 * 4
        ut = torch.zeros((ldr, n), dtype=torch.float64, device="cuda")
        ut[:r] = torch.as_tensor(np.ascontiguousarray(lr.vectors.T), device="cuda")
        aut = torch.zeros_like(ut)
        op.spmm(ut[:r].contiguous(), aut[:r], b=r, chunk=1)
        # A^(m+1) U for the m-term walk start (only the last power is kept)
        powers = [aut]
        for _ in range(self.walk_terms):
            nxt = torch.zeros_like(ut)
            op.spmm(powers[-1][:r].contiguous(), nxt[:r], b=r, chunk=1)
            powers.append(nxt)
        a2ut = powers[1] if self.walk_terms == 1 else None  # powers[k] = A^(k+1) U
        a3ut = powers[2] if self.walk_terms == 2 else None
        a4ut = powers[3] if self.walk_terms == 3 else None
        del powers
        t = ut[:r] @ aut[:r].T
        t = 0.5 * (t + t.T)
        w = torch.linalg.inv(torch.eye(r, dtype=torch.float64, device="cuda") - self.alpha * t)
        self.u = ut.T.contiguous()      # n x ldr row-major
        self.au = aut.T.contiguous()    # n x ldr row-major
        self.w = w.contiguous()
        self.a2u = a2ut.T.contiguous() if a2ut is not None else None  # n x ldr row-major
        self.a3u = a3ut.T.contiguous() if a3ut is not None else None
        self.a4u = a4ut.T.contiguous() if a4ut is not None else None
        self.ritz_values = lr.values.copy()
        self.rank, self.ldr = r, ldr
        del ut, aut, a2ut, a3ut, a4ut
        desc = _lib.KzEigenDesc()
        desc.n, desc.r, desc.ldr = n, r, ldr
        desc.beta = float(self.alpha)
        desc.op = op.handle.value
        desc.u, desc.au, desc.w = self.u.data_ptr(), self.au.data_ptr(), self.w.data_ptr()
        desc.a2u = self.a2u.data_ptr() if self.a2u is not None else None
        desc.a3u = self.a3u.data_ptr() if self.a3u is not None else None
        desc.a4u = self.a4u.data_ptr() if self.a4u is not None else None
        h = ctypes.c_void_p()
        _lib.check(lib.kz_eigen_create(ctypes.byref(desc), ctypes.byref(h)))
        self._lib, self._handle = lib, h
        torch.cuda.synchronize()
        self.build_stats = {"rank": r, "walk_terms": self.walk_terms, "lanczos_seconds": t_lanczos,
                            "build_seconds": time.perf_counter() - t0,
                            "ritz_top": [float(v) for v in lr.values[:4]]}

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                self._lib.kz_eigen_destroy(h)
            except Exception:
                pass
            self._handle = None

    def eigen_handle(self):
        return self._handle

    def basis_internal(self):
        """(U, AU, W) as host arrays with rows in internal node order (U and
        AU live in the GraphIndex's solve order on the device)."""
        r = self.rank
        u = self.u[:, :r].cpu().numpy()
        au = self.au[:, :r].cpu().numpy()
        inv = getattr(self.gi, "_inv", None) if getattr(self.gi, "_order", None) is not None else None
        if inv is not None:
            u, au = u[inv], au[inv]
        return u, au, self.w.cpu().numpy()

    def _internal_rows(self, t):
        if t is None:
            return None
        m = t[:, : self.rank].cpu().numpy()
        inv = getattr(self.gi, "_inv", None) if getattr(self.gi, "_order", None) is not None else None
        return m[inv] if inv is not None else m

    def a2u_internal(self):
        """A^2 U as a host array with rows in internal node order (None
        unless walk_terms == 1)."""
        return self._internal_rows(self.a2u)

    def a3u_internal(self):
        """A^3 U, internal row order (None unless walk_terms == 2)."""
        return self._internal_rows(self.a3u)

    def a4u_internal(self):
        """A^4 U, internal row order (None unless walk_terms == 3)."""
        return self._internal_rows(self.a4u)

    # -- the GraphIndex surface (ids, operator, masks) ----------------------
    @property
    def n(self):
        return self.gi.n

    @property
    def graph(self):
        return self.gi.graph

    def operator(self):
        return self.gi.operator()

    def mask_operator(self):
        return self.gi.mask_operator()

    def solve_positions(self, internal):
        return self.gi.solve_positions(internal)

    def start_vector_to_solve(self, x0):
        return self.gi.start_vector_to_solve(x0)

    def device_perm(self):
        return self.gi.device_perm()

    def internal_id(self, original):
        return self.gi.internal_id(original)

    def internal_ids(self, originals):
        return self.gi.internal_ids(originals)

    def adjacency_internal(self):
        return self.gi.adjacency_internal()

    def rhs_for_position(self, pos):
        return self.gi.rhs_for_position(pos)
