"""Where sparse_katz_batch spends its time at cfg5 (SBM 10^6, s = 100,
T = 101, tol 1e-10): wall time per phase (query solves, top-k, anchor solves,
profile gathers, rerank, host work), anchor-solve iterations and the
deduplication ratio.  python tools/profile_cfg5.py [--queries 128]"""
import argparse
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
from paper_1912_06525_b200 import linkpred, solver

ap = argparse.ArgumentParser()
ap.add_argument("--queries", type=int, default=128)
ap.add_argument("--s", type=int, default=100)
ap.add_argument("--anchor-batch", type=int, default=256)
a = ap.parse_args()

g, pos = G.sbm_split(n=1_000_000, seed=0)
lam = kz.spectral_norm(g)
idx = kz.GraphIndex(g, 0.5 / lam, spectral_norm=lam)
cand = np.unique(pos.ravel())
qs = G.sample_queries(cand, a.queries, seed=0)

acc = {"solve_s": 0.0, "solves": 0, "cols": 0, "iters": []}
orig_qb = solver.query_batch


def timed_qb(index, q, **kw):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = orig_qb(index, q, **kw)
    torch.cuda.synchronize()
    acc["solve_s"] += time.perf_counter() - t
    acc["solves"] += 1
    acc["cols"] += len(q)
    acc["iters"].extend(int(r.iterations) for r in out[1])
    return out


solver.query_batch = timed_qb
kz.sparse_katz_batch(idx, qs[:8], a.s)  # warm-up
acc.update(solve_s=0.0, solves=0, cols=0, iters=[])
torch.cuda.synchronize()
t = time.perf_counter()
kz.sparse_katz_batch(idx, qs, a.s, anchor_batch=a.anchor_batch)
torch.cuda.synchronize()
tot = time.perf_counter() - t
it = np.asarray(acc["iters"])
print(json.dumps({"queries": len(qs), "total_s": round(tot, 3), "solve_s": round(acc["solve_s"], 3),
                  "other_s": round(tot - acc["solve_s"], 3), "solve_calls": acc["solves"],
                  "solved_columns": acc["cols"], "anchor_slots": len(qs) * (a.s + 1),
                  "mean_iterations": round(float(it.mean()), 2), "max_iterations": int(it.max()),
                  "ms_per_column_iteration": round(1e3 * acc["solve_s"] / float(it.sum()), 4),
                  "queries_per_s": round(len(qs) / tot, 1)}))
