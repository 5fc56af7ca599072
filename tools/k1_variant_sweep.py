"""K1 compile-time variant sweep at R-MAT 22 (degree-class + RCM solve order,
b = 256, C = 32): times Y = X - beta*A X with fused dots for one library build
(KZ_LIB_PATH selects it) and checks the result against a saved base result.

  python tools/k1_variant_sweep.py --tag base --save   # first: writes /tmp reference
  KZ_LIB_PATH=build/variants/mb6/libkatzb200.so python tools/k1_variant_sweep.py --tag mb6

The permuted CSR is cached under /tmp so each variant process only pays the
device upload."""
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
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--b", type=int, default=256)
ap.add_argument("--reps", type=int, default=9)
ap.add_argument("--tag", default="base")
ap.add_argument("--save", action="store_true")
ap.add_argument("--cache", default="/tmp/k1sweep")
ap.add_argument("--chunk", type=int, default=32)
a = ap.parse_args()

os.makedirs(a.cache, exist_ok=True)
cf = os.path.join(a.cache, f"csr{a.scale}.npz")
if os.path.exists(cf):
    z = np.load(cf)
    off, col, n, nnz = z["off"], z["col"], int(z["n"]), int(z["nnz"])
else:
    g = G.rmat_graph_fast(a.scale)
    order = degclass_rcm_order(g)
    inv = np.empty(g.n, dtype=np.int64)
    inv[order] = np.arange(g.n)
    off, col = permute_csr(g.row_offsets, g.col_indices, order, inv)
    n, nnz = g.n, g.nnz
    np.savez(cf, off=off, col=col, n=n, nnz=nnz)

b, C = a.b, a.chunk
gen = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(b * n, dtype=torch.float64, device="cuda", generator=gen)
Y = torch.empty_like(X)
dots = torch.empty(b, dtype=torch.float64, device="cuda")
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
rf = os.path.join(a.cache, f"ref{a.scale}_c{C}.pt")
if a.save:
    torch.save({"Y": Y.cpu(), "d": dots.cpu()}, rf)
    err = derr = 0.0
else:
    ref = torch.load(rf)
    Yr, dr = ref["Y"].cuda(), ref["d"].cuda()
    err = float(((Y - Yr).abs().max() / Yr.abs().max()).item())
    derr = float(((dots - dr).abs() / dr.abs()).max().item())
ms = float(np.median(ts))
print(json.dumps({"variant": a.tag, "lib": kz._lib.LIB_PATH if hasattr(kz, "_lib") else None,
                  "ms": round(ms, 3), "ms_min": round(min(ts), 3),
                  "gathered_tbs": round(nnz * 8.0 * b / ms / 1e9, 2),
                  "max_rel_err": err, "dot_rel_err": derr}), flush=True)
