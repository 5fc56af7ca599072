"""Feasibility of the cold-slab split of K1 at R-MAT 22 (b = 256, C = 32,
degree-class + RCM order): entries whose column is outside the L2-resident
hot set (col >= H) are moved, for rows holding at least --min-cold of them,
into virtual rows (slab, row) processed slab-major so each 48 MB slab of X
stays in L2; the main operator keeps the rest.  Times the full operator, the
main operator and the virtual-row operator with the shipped K1 kernel (an
upper bound for a dedicated cold pass, which would not pay a Y row per
virtual row)."""
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
ap.add_argument("--H", type=int, default=131072)
ap.add_argument("--slab-rows", type=int, default=190000)
ap.add_argument("--min-cold", type=int, nargs="+", default=[8, 32])
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--cache", default="/tmp/k1sweep")
a = ap.parse_args()
os.makedirs(a.cache, exist_ok=True)
cf = os.path.join(a.cache, "csr22.npz")
if os.path.exists(cf):
    z = np.load(cf)
    off, col, n = z["off"], z["col"], int(z["n"])
else:
    g = G.rmat_graph_fast(22)
    order = degclass_rcm_order(g)
    inv = np.empty(g.n, dtype=np.int64)
    inv[order] = np.arange(g.n)
    off, col = permute_csr(g.row_offsets, g.col_indices, order, inv)
    n = g.n
    np.savez(cf, off=off, col=col, n=n, nnz=g.nnz)
b, C = 256, 32
X = torch.randn(b * n, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)


def timed(o, c, rows, cols, Yb, xs):
    op = kz.DeviceOperator(o, c.astype(np.int32), rows, cols)
    ts = []
    for r in range(a.reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if xs:
            op.spmm(X, Yb, b=b, chunk=C, Xs=X, s1=1.0, s2=-2e-4)
        else:
            op.spmm(X, Yb, b=b, chunk=C, s2=1.0)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    del op
    return float(np.median(ts))


deg = np.diff(off)
rows = np.repeat(np.arange(n), deg)
full = timed(off, col, n, n, Y, True)
print(json.dumps({"operator": "full", "nnz": int(col.size), "ms": round(full, 3)}), flush=True)
cold = col >= a.H
coldcnt = np.bincount(rows[cold], minlength=n)
for mc in a.min_cold:
    moved = cold & (coldcnt[rows] >= mc)
    # main operator
    keep = ~moved
    oa = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=n), out=oa[1:])
    t_main = timed(oa, col[keep], n, n, Y, True)
    # virtual rows (slab, row), slab-major
    r_m, c_m = rows[moved], col[moved]
    slab = (c_m - a.H) // a.slab_rows
    key = slab.astype(np.int64) * n + r_m
    o = np.argsort(key, kind="stable")
    key, c_s = key[o], c_m[o]
    uk, cnt = np.unique(key, return_counts=True)
    ob = np.zeros(uk.size + 1, dtype=np.int64)
    np.cumsum(cnt, out=ob[1:])
    P = torch.empty(b * uk.size, dtype=torch.float64, device="cuda")
    t_cold = timed(ob, c_s, uk.size, n, P, False)
    del P
    print(json.dumps({"min_cold": mc, "moved_frac": round(float(moved.mean()), 4),
                      "cold_frac": round(float(cold.mean()), 4), "virtual_rows": int(uk.size),
                      "entries_per_virtual_row": round(float(cnt.mean()), 2),
                      "main_ms": round(t_main, 3), "cold_ms": round(t_cold, 3),
                      "sum_ms": round(t_main + t_cold, 3), "full_ms": round(full, 3)}), flush=True)
