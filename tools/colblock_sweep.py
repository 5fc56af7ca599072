"""K1 column-blocking sweep at R-MAT 22 (RCM solve order, b = 256, C = 32):
times Y = X - beta*A X with fused dots for several schedules (env knobs read
by kz_graph_create: KZ_K1_SLICE_MB, KZ_K1_MINDEG, KZ_K1_INTERLEAVE) and checks
each result against the unblocked operator's."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G
from paper_1912_06525_b200.index import permute_csr, rcm_order

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--b", type=int, default=256)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--settings", default="0:128:1,16:128:1,32:128:1,48:128:1,32:64:1,32:1024:1,32:128:0")
ap.add_argument("--out", default=None)
ap.add_argument("--chunk", type=int, default=32)
a = ap.parse_args()

g = G.rmat_graph_fast(a.scale)
order = rcm_order(g)
inv = np.empty(g.n, dtype=np.int64)
inv[order] = np.arange(g.n)
off, col = permute_csr(g.row_offsets, g.col_indices, order, inv)
n, b, C = g.n, a.b, a.chunk
torch.manual_seed(0)
X = torch.randn(b * n, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
Yref = None
dots = torch.empty(b, dtype=torch.float64, device="cuda")
dref = None
rows = []
for s in a.settings.split(","):
    slice_mb, mindeg, inter = s.split(":")
    os.environ["KZ_K1_SLICE_MB"] = slice_mb
    os.environ["KZ_K1_MINDEG"] = mindeg
    os.environ["KZ_K1_INTERLEAVE"] = inter
    op = kz.DeviceOperator(off, col, n)
    ts = []
    for r in range(a.reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        op.spmm(X, Y, b=b, chunk=C, Xs=X, s1=1.0, s2=-2e-4, dots=dots)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    if Yref is None:
        Yref, dref = Y.clone(), dots.clone()
        err = derr = 0.0
    else:
        err = float(((Y - Yref).abs().max() / Yref.abs().max()).item())
        derr = float(((dots - dref).abs() / dref.abs()).max().item())
    ms = float(np.median(ts))
    row = {"slice_mb": float(slice_mb), "min_deg": int(mindeg), "interleave": int(inter), "nseg": op.nitems,
           "ms": round(ms, 3), "ms_min": round(min(ts), 3), "gathered_tbs": round(g.nnz * 8.0 * b / ms / 1e9, 2),
           "max_rel_err": err, "dot_rel_err": derr}
    print(json.dumps(row), flush=True)
    rows.append(row)
    del op
if a.out:
    with open(a.out, "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
