import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G
for cfg in ("cfg1", "proxy16"):
    g = G.config_graph(cfg)
    from paper_1912_06525_b200.graph import device_operator
    op = device_operator(g)
    for b, C in ((16, 16), (64, 32)):
        X = torch.randn(b * g.n, dtype=torch.float64, device="cuda"); Y = torch.empty_like(X)
        dots = torch.empty(b, dtype=torch.float64, device="cuda")
        for dd in (None, dots):
            for _ in range(5): op.spmm(X, Y, b=b, chunk=C, Xs=X, s1=1.0, s2=-1e-3, dots=dd)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(100): op.spmm(X, Y, b=b, chunk=C, Xs=X, s1=1.0, s2=-1e-3, dots=dd)
            e1.record(); torch.cuda.synchronize()
            print(cfg, g.n, g.nnz, "b", b, "dots" if dd is not None else "nodots", round(e0.elapsed_time(e1) / 100 * 1e3, 1), "us")
