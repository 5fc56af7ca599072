"""K1 (C = 32, b = 256) at R-MAT 22 under node orderings aimed at L2 reuse:
RCM (the GraphIndex default), the vertex-separator partition order of the
index build (parts are closed neighbourhoods except for the separator),
hubs first + RCM, and the partition order with a degree-sorted separator.

    python tools/reorder_experiment2.py [scale]
"""
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
from paper_1912_06525_b200.index import permute_csr


def timeit(g, order, b=256, C=32):
    inv = np.empty(g.n, dtype=np.int64)
    inv[order] = np.arange(g.n)
    off, col = permute_csr(g.row_offsets, g.col_indices, order, inv)
    op = kz.DeviceOperator(off, col, g.n)
    X = torch.randn(b * g.n, dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    dots = torch.empty(b, dtype=torch.float64, device="cuda")
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t = time.perf_counter()
        op.spmm(X, Y, b=b, chunk=C, Xs=X, s1=1.0, s2=-1e-4, dots=dots)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    del X, Y, op
    torch.cuda.empty_cache()
    return round(min(ts[1:]) * 1e3, 2)


scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
g = G.rmat_graph_fast(scale)
n = g.n
deg = np.diff(g.row_offsets)
a = sp.csr_matrix((np.ones(g.nnz, dtype=np.int8), g.col_indices, g.row_offsets), shape=(n, n))
rcm = np.asarray(csgraph.reverse_cuthill_mckee(a, symmetric_mode=True), dtype=np.int64)
print("rcm", timeit(g, rcm), flush=True)
for frac in (0.001, 0.01):
    h = int(frac * n)
    hubs = np.argsort(-deg, kind="stable")[:h]
    is_hub = np.zeros(n, bool)
    is_hub[hubs] = True
    order = np.concatenate([hubs, rcm[~is_hub[rcm]]])
    print(f"hubs{frac}+rcm", timeit(g, order), flush=True)
for limit in (4096, 65536):
    t = time.time()
    bp = kz.partition_vertex_separator(g, kz.PartitionConfig(max_part_size=limit))
    tp = time.time() - t
    print(f"partition limit {limit}: n2 {bp.n2} parts {bp.num_parts} in {tp:.1f}s", flush=True)
    print(f"partition{limit}", timeit(g, bp.perm), flush=True)
    sep = bp.perm[bp.n1:]
    sep = sep[np.argsort(-deg[sep], kind="stable")]
    print(f"partition{limit}+sepdeg", timeit(g, np.concatenate([bp.perm[: bp.n1], sep])), flush=True)
    print(f"sepdeg-first+partition{limit}", timeit(g, np.concatenate([sep, bp.perm[: bp.n1]])), flush=True)
