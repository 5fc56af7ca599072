"""Standalone K1 SpMM driver for ncu captures: one config graph, one
Y = X - beta*A X over a b-column block (chunk width C).  Not a benchmark."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--b", type=int, default=64)
ap.add_argument("--chunk", type=int, default=16)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--rcm", action="store_true", help="solve-order operator of GraphIndex (RCM)")
ap.add_argument("--order", default=None, help="GraphIndex reorder mode (rcm | degree)")
a = ap.parse_args()
spec = G.CONFIGS[a.config]
g = G.rmat_graph_fast(spec["scale"]) if spec["kind"] == "rmat" else G.config_graph(a.config)
mode = "rcm" if a.rcm else a.order
op = (kz.GraphIndex(g, 1e-4, reorder=mode).operator() if mode
      else kz.DeviceOperator(g.row_offsets, g.col_indices.astype(np.int32), g.n))
X = torch.randn(a.b * g.n, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
dots = torch.empty(a.b, dtype=torch.float64, device="cuda")
for _ in range(a.reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    op.spmm(X, Y, b=a.b, chunk=a.chunk, Xs=X, s1=1.0, s2=-1e-4, dots=dots)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    gathered = g.nnz * 8.0 * a.b
    print(f"n={g.n} nnz={g.nnz} b={a.b} C={a.chunk} nlong={op.nlong} items={op.nitems} "
          f"{dt*1e3:.3f} ms  gather {gathered/dt/1e12:.2f} TB/s", flush=True)
