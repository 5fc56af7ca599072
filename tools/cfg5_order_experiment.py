"""cfg5 (SBM 10^6): batched plain-CG solve time (256 columns, tol 1e-10) under
the solve orders GraphIndex offers.  python tools/cfg5_order_experiment.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1912_06525_b200 as kz
from paper_1912_06525_b200 import generators as G
from paper_1912_06525_b200 import solver

g, pos = G.sbm_split(n=1_000_000, seed=0)
lam = kz.spectral_norm(g)
cand = np.unique(pos.ravel())
qs = G.sample_queries(cand, 256, seed=0)
for mode in ("none", "rcm", "degclass", "degree"):
    t0 = time.time()
    idx = kz.GraphIndex(g, 0.5 / lam, spectral_norm=lam, reorder=mode)
    ts = []
    for r in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        scores, reps = solver.query_batch(idx, qs, tol=1e-10, device=True)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
        del scores
    it = np.array([r_.iterations for r_ in reps])
    print(json.dumps({"reorder": mode, "solve_ms": round(float(np.median(ts)), 2), "mean_iterations": float(it.mean()),
                      "ms_per_iteration": round(float(np.median(ts)) / float(it.max()), 3),
                      "order_s": round(time.time() - t0, 1)}), flush=True)
    del idx
