"""Query indexes: the reference's KLRC file, and a factor-free graph index.

``load_index`` reads the reference's on-disk KLRC format (index.py:193-333
of the reference; byte layout in SURVEY.md Appendix A) with the same
validation order and error taxonomy: magic, checksum (blake2b-64), version,
then structure.  The result mirrors the reference's ``KatzIndex`` fields.

For the GPU the index is re-expressed once, on first use
(``KatzIndex.device``): the factor reassemblies the reference performs on
every operator application (BlockCholesky.multiply, DenseCholesky.multiply,
index.py:86-91) are exactly ``I - alpha*A`` on the permuted graph, so the
binary pattern of A is recovered from the factors once and uploaded as an
int32 CSR; the LRC operands (per-part inverses, L^-1, U, sigma) are uploaded
by lrc.py.

``GraphIndex`` is the factor-free index for graphs whose LRC index the
reference cannot build (R-MAT 18/22, SBM 10^6): it supports
the plain-CG solver only.
"""

from __future__ import annotations

import hashlib
import os
import struct
import threading
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .factor import BlockCholesky, DenseCholesky, LowRankCorrection
from .graph import Graph, DeviceOperator

MAGIC = b"KLRC"
FORMAT_VERSION = 1


class IndexFormatError(ValueError):
    """The byte stream is not a readable index of this format (index.py:36-37)."""


class IndexMagicError(IndexFormatError):
    """Leading magic bytes are wrong (index.py:40-41)."""


class IndexVersionError(IndexFormatError):
    """Unsupported format version (index.py:44-45)."""


class IndexChecksumError(IndexFormatError):
    """Checksum mismatch: truncated or corrupted (index.py:48-49)."""


@dataclass(frozen=True, eq=False)
class BlockPartition:
    """Interior-then-separator ordering (partition.py:50-79)."""

    perm: np.ndarray
    inv_perm: np.ndarray
    part_boundaries: np.ndarray
    n1: int
    n2: int
    separator_overflow: bool = False

    @property
    def num_parts(self):
        return self.part_boundaries.size - 1

    @property
    def n(self):
        return self.n1 + self.n2

    def separator_nodes(self):
        return self.perm[self.n1 :]


# guards the lazy device uploads below: an index is shared by concurrent
# query threads, and the first callers must not race to create
# (and leak) two copies of one operator
_DEV_LOCK = threading.RLock()


class _DeviceGraphMixin:
    """Lazily uploaded device state shared by both index kinds."""

    def _op_cache(self):
        cache = self.__dict__.get("_dev")
        if cache is None:
            with _DEV_LOCK:
                cache = self.__dict__.setdefault("_dev", {})
        return cache

    def _cached(self, key, make):
        """cache[key], created once under the lock; the upload is complete on
        the device before any thread (on any stream) sees it."""
        cache = self._op_cache()
        val = cache.get(key)
        if val is None:
            with _DEV_LOCK:
                val = cache.get(key)
                if val is None:
                    val = make()
                    from . import _lib

                    _lib.torch_cuda().cuda.current_stream().synchronize()
                    cache[key] = val
        return val

    def internal_id(self, original):
        pos = int(np.searchsorted(self.id_map, original))
        if pos == self.n or self.id_map[pos] != original:
            raise KeyError(f"unknown node id {original}")
        return pos

    def internal_ids(self, originals):
        """Vectorised internal_id; raises KeyError on the first unknown id."""
        o = np.asarray(originals, dtype=np.int64).ravel()
        pos = np.searchsorted(self.id_map, o)
        bad = (pos >= self.n) | (self.id_map[np.minimum(pos, self.n - 1)] != o)
        if np.any(bad):
            raise KeyError(f"unknown node id {int(o[np.flatnonzero(bad)[0]])}")
        return pos.astype(np.int64)


@dataclass(eq=False)
class KatzIndex(_DeviceGraphMixin):
    """Everything needed to answer exact Katz queries (index.py:52-101)."""

    alpha: float
    spectral_norm: float
    bp: BlockPartition
    m12: sp.csr_matrix
    bc: BlockCholesky
    dc: DenseCholesky
    lr: LowRankCorrection
    id_map: np.ndarray
    lanczos_seed: int
    format_version: int = FORMAT_VERSION
    build_stats: dict = field(default=None, repr=False)

    solver_kind = "lrc"

    @property
    def n(self):
        return self.bp.n

    @property
    def n1(self):
        return self.bp.n1

    @property
    def n2(self):
        return self.bp.n2

    # -- the permuted adjacency pattern, recovered from the factors ---------
    def adjacency_permuted(self):
        """CSR (int64 offsets, int64 cols) of A in partition order.

        M = I - alpha*A; the reference reassembles M11 from the part factors
        (factor.py:108-124) and M22 from L (factor.py:180-181) at every
        application.  Off-diagonal entries are -alpha on edges and roundoff
        elsewhere, so thresholding at -alpha/2 recovers A exactly (the same
        rule linkpred._query_state uses on the rhs, linkpred.py:140-141).
        """
        cached = self.__dict__.get("_aperm")
        if cached is not None:
            return cached
        n, n1 = self.n, self.n1
        half = -self.alpha / 2.0
        rows, cols = [], []
        bo = self.bc.block_offsets
        for b in range(self.bc.num_blocks):
            s = int(bo[b])
            lb = self.bc.dense[b]
            if lb.shape[0] < 2:
                continue
            mb = lb @ lb.T
            o = np.asarray(self.bc.orders[b], dtype=np.int64)
            i, j = np.nonzero(mb < half)
            off = i != j
            rows.append(s + o[i[off]])
            cols.append(s + o[j[off]])
        m12 = self.m12.tocoo()
        rows.append(m12.row.astype(np.int64))
        cols.append(m12.col.astype(np.int64) + n1)
        rows.append(m12.col.astype(np.int64) + n1)
        cols.append(m12.row.astype(np.int64))
        if self.n2 > 1:
            m22 = _gram_lower(self.dc.factor)
            i, j = np.nonzero(m22 < half)
            off = i != j
            rows.append(n1 + i[off])
            cols.append(n1 + j[off])
        r = np.concatenate(rows) if rows else np.zeros(0, np.int64)
        c = np.concatenate(cols) if cols else np.zeros(0, np.int64)
        key = np.unique(r * n + c)
        r, c = key // n, key % n
        offsets = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(r, minlength=n), out=offsets[1:])
        self.__dict__["_aperm"] = (offsets, c)
        return offsets, c

    def adjacency_internal(self):
        """CSR of A in internal (graph) order: A_int[perm[i], perm[j]] = A_perm[i, j]."""
        cached = self.__dict__.get("_aint")
        if cached is not None:
            return cached
        off, col = self.adjacency_permuted()
        n = self.n
        perm = self.bp.perm
        row_perm = np.repeat(np.arange(n), np.diff(off))
        r = perm[row_perm]
        c = perm[col]
        key = np.sort(r * n + c)
        r, c = key // n, key % n
        offsets = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(r, minlength=n), out=offsets[1:])
        self.__dict__["_aint"] = (offsets, c)
        return offsets, c

    def operator(self):
        """Device operator of A in partition order (the solve order)."""
        def make():
            off, col = self.adjacency_permuted()
            return DeviceOperator(off, col.astype(np.int32), self.n)
        return self._cached("op", make)

    def mask_operator(self):
        """Device operator of A in internal order (neighbour masks for top-k)."""
        def make():
            off, col = self.adjacency_internal()
            return DeviceOperator(off, col.astype(np.int32), self.n)
        return self._cached("mask", make)

    def solve_positions(self, internal):
        """Positions of internal ids in the solve (partition) order."""
        return self.bp.inv_perm[np.asarray(internal, dtype=np.int64)]

    def device_perm(self):
        def make():
            from . import _lib

            torch = _lib.torch_cuda()
            return torch.as_tensor(self.bp.perm, dtype=torch.int64).cuda()
        return self._cached("perm", make)

    def lrc(self):
        """Device LRC operands (lazily uploaded; see lrc.py)."""
        def make():
            from .lrc import DeviceLRC

            return DeviceLRC(self)
        return self._cached("lrc", make)

    # -- reference methods, evaluated on the device -------------------------
    def apply_m_permuted(self, x):
        """M x = x - alpha*A x in partition order (index.py:86-91)."""
        from .solver import _apply_m_host

        return _apply_m_host(self, x)

    def rhs_for_position(self, pos):
        """alpha * A e_pos in partition order (index.py:93-101)."""
        off, col = self.adjacency_permuted()
        out = np.zeros(self.n)
        out[col[off[pos] : off[pos + 1]]] = self.alpha
        return out


def _gram_lower(lf):
    """L L^T for the dense separator factor (once, at device build)."""
    n = lf.shape[0]
    if n >= 2048:
        try:
            from .lrc import device_gram

            return device_gram(lf)
        except Exception:  # pragma: no cover - no device: numpy BLAS
            pass
    return lf @ lf.T


@dataclass(eq=False)
class GraphIndex(_DeviceGraphMixin):
    """Factor-free index: a graph and its damping factor (plain CG only).

    Used where the reference's LRC build is infeasible; the
    solver is the reference's ``cg`` (solver.py:62-101) on v - alpha*A v
    with rhs alpha*A e_q, i.e. query_cg_baseline in natural order.

    ``reorder`` relabels the nodes *inside the solve* for gather locality
    ("degclass": degree classes, reverse Cuthill-McKee inside each; "rcm";
    "degree"; "auto" = ``auto_order``).  It is invisible at the API:
    right-hand sides, start vectors and scores stay in internal order (the output kernel scatters back); only
    summation order, i.e. roundoff, changes.
    """

    graph: Graph
    alpha: float
    spectral_norm: float = float("nan")
    reorder: str = "auto"

    solver_kind = "cg"

    def __post_init__(self):
        self.id_map = self.graph.original_ids
        g = self.graph
        mode = self.reorder
        self._order = None
        if mode == "auto":
            self._order = auto_order(g)
            mode = None
        if mode == "rcm":
            self._order = rcm_order(g)
        elif mode == "degclass":
            self._order = degclass_rcm_order(g)
        elif mode == "degree":
            self._order = np.argsort(-np.diff(g.row_offsets), kind="stable")
        elif mode not in (None, "none"):
            raise ValueError(f"unknown reorder mode {mode!r}")
        if self._order is not None:
            self._inv = np.empty(g.n, dtype=np.int64)
            self._inv[self._order] = np.arange(g.n)

    @property
    def n(self):
        return self.graph.n

    def operator(self):
        """Device operator in the solve order."""
        def make():
            g = self.graph
            if self._order is None:
                return DeviceOperator(g.row_offsets, g.col_indices.astype(np.int32), g.n)
            off, col = permute_csr(g.row_offsets, g.col_indices, self._order, self._inv)
            return DeviceOperator(off, col, g.n)
        return self._cached("op", make)

    def mask_operator(self):
        """Device operator in internal order (neighbour masks for top-k)."""
        if self._order is None:
            return self.operator()

        def make():
            g = self.graph
            return DeviceOperator(g.row_offsets, g.col_indices.astype(np.int32), g.n)
        return self._cached("mask", make)

    def solve_positions(self, internal):
        internal = np.asarray(internal, dtype=np.int64)
        return internal if self._order is None else self._inv[internal]

    def start_vector_to_solve(self, x0):
        """A start vector given in internal order, in the solve order."""
        return x0 if self._order is None else x0[self._order]

    def device_perm(self):
        if self._order is None:
            return None

        def make():
            from . import _lib

            torch = _lib.torch_cuda()
            return torch.as_tensor(self._order, dtype=torch.int64).cuda()
        return self._cached("perm", make)

    def adjacency_internal(self):
        return self.graph.row_offsets, self.graph.col_indices

    def rhs_for_position(self, pos):
        g = self.graph
        out = np.zeros(g.n)
        out[g.neighbors(pos)] = self.alpha
        return out


def rcm_order(g):
    """Reverse Cuthill-McKee node order (locality of the K1 gathers)."""
    import scipy.sparse.csgraph as csgraph

    a = sp.csr_matrix((np.ones(g.nnz, dtype=np.int8), g.col_indices, g.row_offsets), shape=(g.n, g.n))
    return np.asarray(csgraph.reverse_cuthill_mckee(a, symmetric_mode=True), dtype=np.int64)


def degclass_rcm_order(g):
    """Rows grouped by degree class (floor(log2 deg), highest first), RCM
    order inside each class: rows of similar degree -- which in a power-law
    graph share their hub neighbours -- run together, so K1's gathered rows
    stay in L2 longer (R-MAT 22: K1 18.1 -> 17.4 ms against plain RCM,
    tools/reorder_minhash.py)."""
    rcm = rcm_order(g)
    pos = np.empty(g.n, dtype=np.int64)
    pos[rcm] = np.arange(g.n)
    cls = -np.floor(np.log2(np.maximum(np.diff(g.row_offsets), 1))).astype(np.int64)
    return np.lexsort((pos, cls)).astype(np.int64)


def auto_order(g):
    """Solve order for GraphIndex(reorder="auto"), or None to keep the given
    one.  Operators of at most 10^6 stored entries fit L2 and stay as they are.
    Power-law graphs (max degree above 16x the mean: R-MAT, Chung-Lu) get the
    degree-class order, which keeps the hub rows of X together in L2.  Graphs
    without hubs (the planted-partition graph of BASELINE config 5) gain
    nothing from degree classes; they keep the given order unless RCM brings
    neighbours closer, measured by the median |row - col| over the stored
    entries (SBM 10^6: the generator's community-contiguous ids give 6.06 ms
    per CG iteration at 256 columns, RCM 6.65, degree classes 6.76;
    tools/cfg5_order_experiment.py)."""
    if g.nnz <= 1_000_000:
        return None
    deg = np.diff(g.row_offsets)
    if deg.max() > 16.0 * deg.mean():
        return degclass_rcm_order(g)
    rows = np.repeat(np.arange(g.n, dtype=np.int64), deg)
    cols = np.asarray(g.col_indices, dtype=np.int64)
    rcm = rcm_order(g)
    pos = np.empty(g.n, dtype=np.int64)
    pos[rcm] = np.arange(g.n)
    gap_given = np.median(np.abs(rows - cols))
    gap_rcm = np.median(np.abs(pos[rows] - pos[cols]))
    return None if gap_given <= gap_rcm else rcm


def permute_csr(offsets, cols, order, inv):
    """Rows/cols relabelled: new row i = old row order[i], new col = inv[old col].
    Column order within a row is kept (K1 does not need sorted rows)."""
    deg = np.diff(offsets)[order]
    new_off = np.zeros(order.size + 1, dtype=np.int64)
    np.cumsum(deg, out=new_off[1:])
    src = np.repeat(offsets[order] - new_off[:-1], deg) + np.arange(new_off[-1], dtype=np.int64)
    return new_off, inv[cols[src]].astype(np.int32)


# ---------------------------------------------------------------------------
# KLRC reader / writer (layout: SURVEY.md Appendix A)
# ---------------------------------------------------------------------------


class _Cursor:
    def __init__(self, buf):
        self.buf = buf
        self.pos = 0

    def raw(self, nbytes, what):
        end = self.pos + nbytes
        if nbytes < 0 or end > len(self.buf):
            raise IndexFormatError(f"stream ended inside {what}")
        out = self.buf[self.pos : end]
        self.pos = end
        return out

    def i64(self, count, what):
        return np.frombuffer(self.raw(8 * count, what), dtype="<i8").astype(np.int64)

    def f64(self, count, what):
        return np.frombuffer(self.raw(8 * count, what), dtype="<f8").astype(np.float64)

    def u64(self, what):
        return struct.unpack("<Q", self.raw(8, what))[0]

    def csr(self, nrows, ncols, what):
        nnz = self.u64(what)
        indptr = self.i64(nrows + 1, what)
        indices = self.i64(nnz, what)
        data = self.f64(nnz, what)
        if indptr[0] != 0 or indptr[-1] != nnz or np.any(np.diff(indptr) < 0):
            raise IndexFormatError(f"bad CSR offsets in {what}")
        if nnz and (indices.min() < 0 or indices.max() >= ncols):
            raise IndexFormatError(f"column index out of range in {what}")
        return sp.csr_matrix((data, indices, indptr), shape=(nrows, ncols))


def load_index(source):
    """Read a KLRC index (index.py:261-333 semantics; checks magic, checksum,
    version, then structure)."""
    if isinstance(source, (str, os.PathLike)):
        with open(source, "rb") as fh:
            data = fh.read()
    else:
        data = source.read()
    if len(data) < 4 or data[:4] != MAGIC:
        raise IndexMagicError("not an index file (bad magic)")
    if len(data) < 17:
        raise IndexChecksumError("stream truncated")
    if hashlib.blake2b(data[:-8], digest_size=8).digest() != data[-8:]:
        raise IndexChecksumError("checksum mismatch; file truncated or corrupted")
    version, flags = struct.unpack_from("<IB", data, 4)
    if version != FORMAT_VERSION:
        raise IndexVersionError(f"unsupported index version {version}")
    cur = _Cursor(memoryview(data)[:-8])
    cur.pos = 9
    alpha, norm = struct.unpack("<dd", cur.raw(16, "header"))
    seed, n, n1, n2, ell, num_parts = struct.unpack("<6Q", cur.raw(48, "header"))
    if n1 + n2 != n:
        raise IndexFormatError("inconsistent block sizes")
    id_map = cur.i64(n, "id map")
    perm = cur.i64(n, "permutation")
    bounds = cur.i64(num_parts + 1, "part boundaries")
    if bounds[0] != 0 or bounds[-1] != n1 or np.any(np.diff(bounds) < 0):
        raise IndexFormatError("bad part boundaries")
    if not np.array_equal(np.sort(perm), np.arange(n)):
        raise IndexFormatError("permutation is not a permutation")
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    m12 = cur.csr(n1, n2, "coupling block")
    orders, factors = [], []
    for b in range(num_parts):
        size = int(bounds[b + 1] - bounds[b])
        order = cur.i64(size, f"part {b} ordering")
        if not np.array_equal(np.sort(order), np.arange(size)):
            raise IndexFormatError(f"part {b} ordering is not a permutation")
        orders.append(order)
        factors.append(cur.csr(size, size, f"part {b} factor"))
    lfac = cur.f64(n2 * n2, "separator factor").reshape((n2, n2), order="F")
    vecs = cur.f64(n2 * ell, "correction vectors").reshape((n2, ell), order="F")
    vals = cur.f64(ell, "correction values")
    if cur.pos != len(cur.buf):
        raise IndexFormatError("trailing bytes after payload")
    bp = BlockPartition(perm=perm, inv_perm=inv, part_boundaries=bounds, n1=int(n1), n2=int(n2),
                        separator_overflow=bool(flags & 1))
    return KatzIndex(
        alpha=alpha,
        spectral_norm=norm,
        bp=bp,
        m12=m12,
        bc=BlockCholesky(block_offsets=bounds, orders=orders, factors=factors),
        dc=DenseCholesky(factor=lfac),
        lr=LowRankCorrection(ell=int(ell), vectors=vecs, values=vals),
        id_map=id_map,
        lanczos_seed=int(seed),
        format_version=int(version),
    )


def save_index(idx, sink):
    """Write a KatzIndex in the KLRC layout (index.py:193-225 semantics)."""
    parts = [MAGIC, struct.pack("<IB", idx.format_version, 1 if idx.bp.separator_overflow else 0),
             struct.pack("<dd", idx.alpha, idx.spectral_norm),
             struct.pack("<6Q", idx.lanczos_seed, idx.n, idx.n1, idx.n2, idx.lr.ell, idx.bp.num_parts)]

    def ints(a):
        parts.append(np.ascontiguousarray(a, dtype="<i8").tobytes())

    def csr(m):
        parts.append(struct.pack("<Q", m.nnz))
        ints(m.indptr)
        ints(m.indices)
        parts.append(np.asarray(m.data, dtype="<f8").tobytes())

    ints(idx.id_map)
    ints(idx.bp.perm)
    ints(idx.bp.part_boundaries)
    csr(idx.m12)
    for b in range(idx.bc.num_blocks):
        ints(idx.bc.orders[b])
        csr(idx.bc.factors[b])
    parts.append(np.asarray(idx.dc.factor, dtype="<f8").tobytes(order="F"))
    parts.append(np.asarray(idx.lr.vectors, dtype="<f8").tobytes(order="F"))
    parts.append(np.asarray(idx.lr.values, dtype="<f8").tobytes())
    payload = b"".join(parts)
    blob = payload + hashlib.blake2b(payload, digest_size=8).digest()
    if isinstance(sink, (str, os.PathLike)):
        with open(sink, "wb") as fh:
            fh.write(blob)
    else:
        sink.write(blob)
