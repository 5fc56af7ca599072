"""K1 alone on the cfg5 graph (SBM 10^6, given order): Y = X - beta*A X with
fused dots at b = 256, C = 32, and the streaming floor of the same launch
(an operator with no entries: epilogue streams only)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G

g, _ = G.sbm_split(n=1_000_000, seed=0)
n, b, C = g.n, 256, int(os.environ.get("K1_C", "32"))
X = torch.randn(b * n, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
Z = torch.randn(b * n, dtype=torch.float64, device="cuda")
dots = torch.empty(b, dtype=torch.float64, device="cuda")


def timed(op, **kw):
    ts = []
    for r in range(9):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.spmm(X, Y, b=b, chunk=C, Xs=X, s1=1.0, s2=-2e-2, dots=dots, **kw)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    return round(float(np.median(ts)), 3)


op = kz.DeviceOperator(g.row_offsets, g.col_indices.astype(np.int32), n)
empty = kz.DeviceOperator(np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int32), n)
deg = np.diff(g.row_offsets)
print(json.dumps({"C": C, "n": n, "nnz": int(g.nnz), "max_deg": int(deg.max()),
                  "k1_ms": timed(op), "k1_with_z_ms": timed(op, Z=Z, s0=0.5),
                  "epilogue_only_ms": timed(empty), "gathered_gb": round(g.nnz * 8.0 * b / 1e9, 2),
                  "stream_gb": round(3 * 8.0 * n * b / 1e9, 2)}))
