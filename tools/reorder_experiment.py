"""K1 time at cfg3 under different node orderings (locality experiment)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
import scipy.sparse.csgraph as csgraph
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G


def permuted(g, order):
    """relabel: new id i = old id order[i]"""
    n = g.n
    inv = np.empty(n, dtype=np.int64)
    inv[order] = np.arange(n)
    a = sp.csr_matrix((np.ones(g.nnz, dtype=np.int8), g.col_indices, g.row_offsets), shape=(n, n))
    b = a[order][:, order].tocsr()
    b.sort_indices()
    return b.indptr.astype(np.int64), b.indices.astype(np.int32)


def timeit(off, col, n, b=256, C=16):
    op = kz.DeviceOperator(off, col, n)
    X = torch.randn(b * n, dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    dots = torch.empty(b, dtype=torch.float64, device="cuda")
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        op.spmm(X, Y, b=b, chunk=C, Xs=X, s1=1.0, s2=-1e-4, dots=dots)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best * 1e3


scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
g = G.rmat_graph_fast(scale)
n = g.n
deg = np.diff(g.row_offsets)
print("original", timeit(g.row_offsets, g.col_indices.astype(np.int32), n), flush=True)
order = np.argsort(-deg, kind="stable")
print("degree-desc", timeit(*permuted(g, order), n), flush=True)
a = sp.csr_matrix((np.ones(g.nnz, dtype=np.int8), g.col_indices, g.row_offsets), shape=(n, n))
t = time.time()
bfs = csgraph.breadth_first_order(a, int(np.argmax(deg)), directed=False, return_predecessors=False)
print("bfs order time", time.time() - t, flush=True)
print("bfs", timeit(*permuted(g, bfs), n), flush=True)
t = time.time()
rcm = csgraph.reverse_cuthill_mckee(a, symmetric_mode=True)
print("rcm order time", time.time() - t, flush=True)
print("rcm", timeit(*permuted(g, np.asarray(rcm)), n), flush=True)
