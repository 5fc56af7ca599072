"""K1 time split by row class: only short rows (deg <= 32) vs only longer rows."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G


def t_spmm(off, col, n, X, Y, b=256, C=16):
    op = kz.DeviceOperator(off, col, n)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        op.spmm(X, Y, b=b, chunk=C, Xs=X, s1=1.0, s2=-1e-4)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best * 1e3


g = G.rmat_graph_fast(22)
n = g.n
X = torch.randn(256 * n, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
col = g.col_indices.astype(np.int32)
deg = np.diff(g.row_offsets)
rows = np.repeat(np.arange(n), deg)
print(f"full {t_spmm(g.row_offsets, col, n, X, Y):.2f} ms", flush=True)
for name, keep_row in (("short<=32", deg <= 32), ("long>32", deg > 32)):
    m = keep_row[rows]
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.where(keep_row, deg, 0), out=off[1:])
    ms = t_spmm(off, col[m], n, X, Y)
    print(f"{name}: rows={int(keep_row.sum())} nnz={int(m.sum())} {ms:.2f} ms  gather {m.sum()*8*256/ms/1e9:.2f} TB/s", flush=True)
