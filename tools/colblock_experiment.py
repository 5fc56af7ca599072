"""Does restricting K1 to a column range (L2-resident X slice) raise the
gather rate?  Times A[:, range_k] X for K column ranges vs the full A."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G


def t_spmm(off, col, n, X, Y, b=256, C=16, Z=None):
    op = kz.DeviceOperator(off, col, n)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        op.spmm(X, Y, b=b, chunk=C, Z=Z, s0=1.0, s2=-1e-4)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best * 1e3


g = G.rmat_graph_fast(22)
n = g.n
X = torch.randn(256 * n, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
col = g.col_indices.astype(np.int32)
full = t_spmm(g.row_offsets, col, n, X, Y)
print(f"full nnz={g.nnz} {full:.2f} ms  gather {g.nnz*8*256/full/1e9:.2f} TB/s", flush=True)
rows = np.repeat(np.arange(n), np.diff(g.row_offsets))
for K in (2, 3, 4):
    tot = 0.0
    bounds = np.linspace(0, n, K + 1).astype(np.int64)
    for k in range(K):
        m = (col >= bounds[k]) & (col < bounds[k + 1])
        off = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows[m], minlength=n), out=off[1:])
        ms = t_spmm(off, col[m], n, X, Y, Z=Y if k else None)
        tot += ms
        print(f"  K={K} range {k}: nnz={int(m.sum())} {ms:.2f} ms  gather {m.sum()*8*256/ms/1e9:.2f} TB/s", flush=True)
    print(f"K={K} total {tot:.2f} ms", flush=True)
