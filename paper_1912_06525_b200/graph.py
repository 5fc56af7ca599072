"""Graphs in CSR form, the reference's graph rules, and the device operator.

Host-side ingestion mirrors lrckatz.graph (graph.py:39-326): the same CSR
invariants (symmetric, sorted columns, no self loops or duplicates,
``original_ids`` strictly increasing), the same largest-component rule and
the same spectral-norm estimator.  Ingestion is not the hot path; it only
produces the operator that ``DeviceOperator`` uploads once (int32 column
indices, no stored values) for the sm_100a kernels.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib


class GraphParseError(ValueError):
    """Malformed edge-list input; carries the 1-based line number (graph.py:17-24)."""

    def __init__(self, message, line_no=None):
        if line_no is not None:
            message = f"line {line_no}: {message}"
        super().__init__(message)
        self.line_no = line_no


class ConvergenceError(RuntimeError):
    """Iteration budget exhausted; ``estimate`` holds the last value (graph.py:27-32)."""

    def __init__(self, message, estimate):
        super().__init__(message)
        self.estimate = estimate


class InadmissibleAlphaError(ValueError):
    """Damping factor outside (0, 1/spectral_norm) (graph.py:35-36)."""


@dataclass(frozen=True, eq=False)
class Graph:
    """Undirected graph in CSR form (graph.py:39-108)."""

    n: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    original_ids: np.ndarray

    @property
    def num_edges(self):
        return self.col_indices.size // 2

    @property
    def nnz(self):
        return int(self.col_indices.size)

    def degree(self, u):
        return int(self.row_offsets[u + 1] - self.row_offsets[u])

    def degrees(self):
        return np.diff(self.row_offsets)

    def neighbors(self, u):
        return self.col_indices[self.row_offsets[u] : self.row_offsets[u + 1]]

    def internal_id(self, original):
        pos = int(np.searchsorted(self.original_ids, original))
        if pos == self.n or self.original_ids[pos] != original:
            raise KeyError(f"unknown node id {original}")
        return pos

    def adjacency(self):
        import scipy.sparse as sp

        return sp.csr_matrix(
            (np.ones(self.col_indices.size), self.col_indices, self.row_offsets),
            shape=(self.n, self.n),
        )


def csr_from_pairs(u, v, n):
    """Symmetric, deduplicated, loop-free CSR from endpoint arrays.

    Same result as from_edges (graph.py:111-148): columns sorted within each
    row.  Vectorised: one sort of the directed keys src*n+dst.
    """
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    keep = u != v
    u, v = u[keep], v[keep]
    lo = np.minimum(u, v)
    hi = np.maximum(u, v)
    und = np.unique(lo * n + hi)
    lo, hi = und // n, und % n
    del und
    keys = np.concatenate([lo * n + hi, hi * n + lo])
    del lo, hi
    keys.sort(kind="stable")
    src = keys // n
    dst = keys % n
    del keys
    counts = np.bincount(src, minlength=n)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return offsets, dst


def from_edges(edges, n=None, original_ids=None):
    """Build a Graph from (u, v) internal-id pairs (graph.py:111-148)."""
    arr = np.asarray(edges if isinstance(edges, np.ndarray) else list(edges), dtype=np.int64)
    if arr.size == 0:
        arr = arr.reshape(0, 2)
    if arr.ndim != 2 or arr.shape[1] != 2:
        raise ValueError("edges must be (m, 2)")
    if n is None:
        if arr.size == 0:
            raise ValueError("cannot infer node count from empty edge set")
        n = int(arr.max()) + 1
    if arr.size and (arr.min() < 0 or arr.max() >= n):
        raise ValueError("edge endpoint out of range")
    offsets, dst = csr_from_pairs(arr[:, 0], arr[:, 1], n)
    if original_ids is None:
        original_ids = np.arange(n, dtype=np.int64)
    else:
        original_ids = np.asarray(original_ids, dtype=np.int64)
        if original_ids.shape != (n,):
            raise ValueError("original_ids has wrong length")
    return Graph(n=n, row_offsets=offsets, col_indices=dst, original_ids=original_ids)


def largest_connected_component(g):
    """Largest component, ties to the one holding the smallest original id
    (graph.py:232-261); internal ids relabelled in increasing order."""
    if g.n == 0:
        raise ValueError("empty graph")
    import scipy.sparse.csgraph as csgraph

    count, labels = csgraph.connected_components(g.adjacency(), directed=False)
    if count == 1:
        return g
    sizes = np.bincount(labels, minlength=count)
    # the reference numbers components by their smallest node; pick, among the
    # largest ones, the component whose smallest node is smallest
    first = np.full(count, g.n, dtype=np.int64)
    np.minimum.at(first, labels, np.arange(g.n))
    cands = np.flatnonzero(sizes == sizes.max())
    best = cands[np.argmin(first[cands])]
    keep = np.flatnonzero(labels == best)
    remap = np.full(g.n, -1, dtype=np.int64)
    remap[keep] = np.arange(keep.size)
    deg = np.diff(g.row_offsets)[keep]
    offsets = np.zeros(keep.size + 1, dtype=np.int64)
    np.cumsum(deg, out=offsets[1:])
    # a component is closed under adjacency, so its rows keep every column
    row_of = np.repeat(np.arange(g.n), np.diff(g.row_offsets))
    mask = labels[row_of] == best
    cols = remap[g.col_indices[mask]]
    return Graph(n=int(keep.size), row_offsets=offsets, col_indices=cols,
                 original_ids=g.original_ids[keep].copy())


def load_edge_list(source, fmt="auto"):
    """Read an undirected edge list into a Graph (graph.py:157-208).

    source: path, bytes or file-like; one edge per line, two non-negative
    integer ids separated by whitespace or a comma ("auto": a line holding a
    comma is CSV); blank lines and '#' comments are skipped.  Ids are
    compacted to 0..n-1 in increasing order and kept as original_ids;
    duplicates and self loops are dropped.  GraphParseError (with the line
    number) on a malformed line or when no edge remains.  Parsing is host
    text processing; the CSR is then built like from_edges.
    """
    # like the reference, any fmt other than "csv" / "auto" splits on whitespace (no validation)
    if isinstance(source, (str, os.PathLike)):
        with open(source, "rb") as fh:
            data = fh.read()
    elif isinstance(source, bytes):
        data = source
    else:
        data = source.read()
        if isinstance(data, str):
            data = data.encode()
    us, vs = [], []
    for line_no, raw in enumerate(data.decode("utf-8", errors="replace").splitlines(), 1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        if fmt == "csv" or (fmt == "auto" and "," in line):
            toks = [t.strip() for t in line.split(",") if t.strip()]
        else:
            toks = line.split()
        if len(toks) != 2:
            raise GraphParseError(f"expected 2 fields, got {len(toks)}", line_no)
        try:
            u, v = int(toks[0]), int(toks[1])
        except ValueError:
            raise GraphParseError(f"non-integer node id in {toks!r}", line_no) from None
        if u < 0 or v < 0:
            raise GraphParseError("negative node id", line_no)
        if u != v:
            us.append(u)
            vs.append(v)
    if not us:
        raise GraphParseError("no edges in input")
    arr = np.stack([np.asarray(us, dtype=np.int64), np.asarray(vs, dtype=np.int64)], axis=1)
    ids = np.unique(arr)
    return from_edges(np.searchsorted(ids, arr), n=ids.size, original_ids=ids)


def from_edges_device(u, v, n, original_ids=None):
    """from_edges (graph.py:111-148) on the GPU through kz_edges_to_csr (radix
    sort of the undirected keys, unique, directed expansion, second sort):
    the same CSR (symmetric, deduplicated, loop-free, columns sorted within
    rows).  u, v: int64 endpoint arrays (numpy or torch).  Returns a host
    Graph plus the device CSR (offsets int64, columns int32, rows int32) for
    chaining."""
    torch = _lib.torch_cuda()
    lib = _lib.load()
    ut = torch.as_tensor(u, dtype=torch.int64).cuda().contiguous()
    vt = torch.as_tensor(v, dtype=torch.int64).cuda().contiguous()
    m = int(ut.numel())
    if int(vt.numel()) != m:
        raise ValueError("endpoint arrays differ in length")
    off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    cap = max(2 * m, 1)
    dst = torch.empty(cap, dtype=torch.int32, device="cuda")
    src = torch.empty(cap, dtype=torch.int32, device="cuda")
    nnz = ctypes.c_int64(0)
    ws = torch.empty(max(int(lib.kz_edges_to_csr_workspace_bytes(n, m)), 256), dtype=torch.uint8, device="cuda")
    _lib.check(lib.kz_edges_to_csr(n, m, _lib.ptr(ut), _lib.ptr(vt), _lib.ptr(off), _lib.ptr(dst), _lib.ptr(src),
                                   ctypes.byref(nnz), _lib.ptr(ws), ws.numel(), _lib.stream_ptr(torch)))
    del ws, ut, vt
    dst, src = dst[: nnz.value], src[: nnz.value]
    if original_ids is None:
        original_ids = np.arange(n, dtype=np.int64)
    g = Graph(n=n, row_offsets=off.cpu().numpy(), col_indices=dst.cpu().numpy().astype(np.int64),
              original_ids=np.asarray(original_ids, dtype=np.int64))
    return g, (off, dst, src)


def largest_connected_component_device(g, dev=None):
    """largest_connected_component (graph.py:232-261) with the components
    computed by kz_connected_components (hook + pointer jumping, labels =
    smallest node id) and the relabelled CSR built on the device."""
    torch = _lib.torch_cuda()
    lib = _lib.load()
    n = g.n
    if dev is None:
        off = torch.as_tensor(g.row_offsets, dtype=torch.int64).cuda()
        dst = torch.as_tensor(g.col_indices, dtype=torch.int32).cuda()
        src = torch.repeat_interleave(torch.arange(n, device="cuda", dtype=torch.int32), off[1:] - off[:-1])
    else:
        off, dst, src = dev
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    s32 = src.to(torch.int32).contiguous()
    d32 = dst.to(torch.int32).contiguous()
    _lib.check(lib.kz_connected_components(n, int(d32.numel()), _lib.ptr(s32), _lib.ptr(d32), _lib.ptr(labels),
                                           _lib.stream_ptr(torch)))
    lab = labels.to(torch.int64)
    sizes = torch.bincount(lab, minlength=n)
    big = int(sizes.max().item())
    if big == n:
        return g
    # largest size; ties -> the component whose smallest id (its label) is smallest
    best = int(torch.nonzero(sizes == big)[0].item())
    keep = torch.nonzero(lab == best).flatten()
    remap = torch.full((n,), -1, dtype=torch.int64, device="cuda")
    remap[keep] = torch.arange(keep.numel(), device="cuda")
    mask = lab[src.long()] == best
    cols = remap[dst[mask].long()]
    deg = (off[1:] - off[:-1])[keep]
    new_off = torch.zeros(keep.numel() + 1, dtype=torch.int64, device="cuda")
    new_off[1:] = torch.cumsum(deg, 0)
    keep_h = keep.cpu().numpy()
    return Graph(n=int(keep.numel()), row_offsets=new_off.cpu().numpy(), col_indices=cols.cpu().numpy(),
                 original_ids=g.original_ids[keep_h].copy())


def hardest_alpha(norm):
    """1/(norm + 1) (graph.py:300-308)."""
    if norm < 0:
        raise ValueError("spectral norm must be nonnegative")
    return 1.0 / (norm + 1.0)


@dataclass(frozen=True)
class KatzParams:
    """Validated (alpha, spectral_norm) pair (graph.py:311-326)."""

    alpha: float
    spectral_norm: float

    def __post_init__(self):
        if not (self.alpha > 0.0) or not (self.alpha * self.spectral_norm < 1.0):
            raise InadmissibleAlphaError(
                f"alpha={self.alpha} outside (0, 1/{self.spectral_norm})"
            )


class DeviceOperator:
    """A binary CSR pattern resident on the GPU (kz_graph handle).

    rows x cols pattern; rowptr int64[rows+1], colidx int32[nnz] (numpy or
    torch CUDA tensors).  Immutable; freed with the object.
    """

    def __init__(self, rowptr, colidx, rows, cols=None):
        lib = _lib.load()
        self._lib = lib
        self.rows = int(rows)
        self.cols = int(rows if cols is None else cols)
        keep = []
        if isinstance(rowptr, np.ndarray):
            rp = np.ascontiguousarray(rowptr, dtype=np.int64)
            keep.append(rp)
            rp_ptr = ctypes.c_void_p(rp.ctypes.data)
            nnz = int(rp[-1])
        else:
            rp = rowptr.contiguous()
            keep.append(rp)
            rp_ptr = ctypes.c_void_p(rp.data_ptr())
            nnz = int(rp[-1].item())
        if isinstance(colidx, np.ndarray):
            ci = np.ascontiguousarray(colidx, dtype=np.int32)
            keep.append(ci)
            ci_ptr = ctypes.c_void_p(ci.ctypes.data)
        else:
            ci = colidx.contiguous()
            keep.append(ci)
            ci_ptr = ctypes.c_void_p(ci.data_ptr())
        _lib.torch_cuda()  # a device must exist
        h = ctypes.c_void_p()
        _lib.check(lib.kz_graph_create(self.rows, self.cols, nnz, rp_ptr, ci_ptr, ctypes.byref(h)))
        self.handle = h
        self.nnz = nnz
        vals = [ctypes.c_int64() for _ in range(5)]
        _lib.check(lib.kz_graph_info(h, *[ctypes.byref(v) for v in vals]))
        self.nlong = vals[3].value
        self.nitems = vals[4].value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.kz_graph_destroy(h)
            except Exception:
                pass
            self.handle = None

    def spmm(self, Xg, Y, *, b, chunk=1, Xs=None, Z=None, s0=0.0, s1=0.0, s2=1.0, D=None, dots=None):
        """Y = s0*Z + s1*Xs + s2*(A Xg) on device blocks (layout [b/C][.][C])."""
        torch = _lib.torch_cuda()
        nbytes = self._lib.kz_spmm_workspace_bytes(self.handle, b, chunk)
        ws = _lib.Workspace.get(torch, nbytes, slot="spmm")
        _lib.check(
            self._lib.kz_spmm(
                self.handle, b, chunk, _lib.ptr(Xg), _lib.ptr(Xs), _lib.ptr(Z), _lib.ptr(Y),
                float(s0), float(s1), float(s2), _lib.ptr(D), _lib.ptr(dots),
                _lib.ptr(ws), ws.numel(), _lib.stream_ptr(torch),
            )
        )
        return Y


def device_operator(g):
    """Upload a Graph's adjacency pattern (natural order)."""
    return DeviceOperator(g.row_offsets, g.col_indices.astype(np.int32, copy=False), g.n)


def spectral_norm(g, tol=1e-7, max_iter=10000, op=None):
    """Largest |eigenvalue| of A by power iteration on A@A (graph.py:264-297),
    with both products run by the K1 SpMM on the device."""
    if g.n == 0:
        raise ValueError("empty graph")
    if g.col_indices.size == 0:
        return 0.0
    torch = _lib.torch_cuda()
    lib = _lib.load()
    op = op or device_operator(g)
    n = g.n
    v = torch.full((n,), 1.0 / np.sqrt(n), dtype=torch.float64, device="cuda")
    t = torch.empty_like(v)
    w = torch.empty_like(v)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    st = _lib.stream_ptr(torch)

    def dot(x, y):
        _lib.coldot(torch, lib, x, y, out, n, 1, st)
        return float(out.item())

    last = 0.0
    for _ in range(max_iter):
        op.spmm(v, t, b=1)
        op.spmm(t, w, b=1)
        est = np.sqrt(dot(v, w))
        nw = np.sqrt(dot(w, w))
        if nw == 0.0:
            return 0.0
        _lib.vec_op(torch, lib, 1, n, nw, w, 0.0, None, v)  # v = w / nw
        if abs(est - last) <= tol * max(est, 1e-300):
            op.spmm(v, t, b=1)
            return float(np.sqrt(dot(t, t)))
        last = est
    raise ConvergenceError(
        f"spectral norm estimate did not settle in {max_iter} iterations", float(last)
    )
