"""Can the HBM-bound CG vector updates hide under the L2/LSU-bound K1?
Times, at R-MAT 22 (RCM order, 128 columns = 4 chunks of 32): K1 alone, a
streaming update of the other half-batch's vectors alone (torch, ~K2's bytes:
r -= a*q then p = r + b*p on 2.45 GB blocks), and both launched together on
two streams.  Run with KZ_K1_CTAS=4 / 5 to leave (or not) an SM slot free."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G
from paper_1912_06525_b200.index import permute_csr, rcm_order

g = G.rmat_graph_fast(22)
order = rcm_order(g)
inv = np.empty(g.n, dtype=np.int64)
inv[order] = np.arange(g.n)
off, col = permute_csr(g.row_offsets, g.col_indices, order, inv)
op = kz.DeviceOperator(off, col, g.n)
n, b = g.n, 128
X = torch.randn(b * n, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
dots = torch.empty(b, dtype=torch.float64, device="cuda")
r = torch.randn(b * n, dtype=torch.float64, device="cuda")
q = torch.randn(b * n, dtype=torch.float64, device="cuda")
p = torch.randn(b * n, dtype=torch.float64, device="cuda")
x = torch.randn(b * n, dtype=torch.float64, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def k1():
    op.spmm(X, Y, b=b, chunk=32, Xs=X, s1=1.0, s2=-2e-4, dots=dots)


def k2():
    r.sub_(q, alpha=0.3)
    x.add_(p, alpha=0.2)
    p.mul_(0.1).add_(r)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    ev = torch.cuda.Event()
    ev.record()
    sa.wait_event(ev)
    sb.wait_event(ev)
    with torch.cuda.stream(sa):
        k1()
    with torch.cuda.stream(sb):
        k2()
    torch.cuda.current_stream().wait_stream(sa)
    torch.cuda.current_stream().wait_stream(sb)


t1, t2, t12 = timed(k1), timed(k2), timed(both)
print(f"KZ_K1_CTAS={os.environ.get('KZ_K1_CTAS', '5')}: K1(128 cols) {t1:.2f} ms, stream update {t2:.2f} ms, "
      f"sum {t1 + t2:.2f} ms, concurrent {t12:.2f} ms", flush=True)
