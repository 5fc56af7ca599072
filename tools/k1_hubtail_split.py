"""How K1's time splits between hub and tail columns at R-MAT 22 (b = 256,
C = 32, the bench's degree-class + RCM solve order, where the columns of
highest degree come first): times the full operator and the two operators
holding only the entries whose column is below / at or above H.

  python tools/k1_hubtail_split.py [--H 131072 ...]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G
from paper_1912_06525_b200.index import degclass_rcm_order, permute_csr

ap = argparse.ArgumentParser()
ap.add_argument("--H", type=int, nargs="+", default=[32768, 131072, 524288])
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
g = G.rmat_graph_fast(22)
order = degclass_rcm_order(g)
inv = np.empty(g.n, dtype=np.int64)
inv[order] = np.arange(g.n)
off, col = permute_csr(g.row_offsets, g.col_indices, order, inv)
n, b, C = g.n, 256, 32
X = torch.randn(b * n, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)


def timed(o, c):
    op = kz.DeviceOperator(o, c.astype(np.int32), n)
    for _ in range(2):
        op.spmm(X, Y, b=b, chunk=C, Xs=X, s1=1.0, s2=-2e-4)
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.spmm(X, Y, b=b, chunk=C, Xs=X, s1=1.0, s2=-2e-4)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    del op
    return float(np.median(ts))


rows = np.repeat(np.arange(n), np.diff(off))
full = timed(off, col)
print(json.dumps({"operator": "full", "nnz": int(len(col)), "ms": full}), flush=True)
for H in a.H:
    for name, keep in (("hub", col < H), ("tail", col >= H)):
        r, c = rows[keep], col[keep]
        o = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(r, minlength=n), out=o[1:])
        ms = timed(o, c)
        print(json.dumps({"operator": name, "H": H, "nnz": int(keep.sum()), "frac_nnz": round(float(keep.mean()), 3),
                          "ms": round(ms, 3), "frac_of_full_time": round(ms / full, 3)}), flush=True)
