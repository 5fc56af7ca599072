"""cfg5: modularity-based link-prediction scoring (sparse_katz) on the planted
partition graph (SBM n=10^6, 1,000 power-law communities, mean degree 20,
10% of edges held out), beta=0.5/lambda, s=100, T=101, tol 1e-10
(linkpred default).  Prints queries/s of sparse_katz_batch, the number of
(deduplicated) anchor solves, recall@100 of the reranked lists against the
held-out edges (a sanity signal, not a parity check), and --check N queries
against the CPU oracle restatement (linkpred.py:165-207 over the CSR cg)."""
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

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--queries", type=int, default=1024)
ap.add_argument("--s", type=int, default=100)
ap.add_argument("--check", type=int, default=1)
ap.add_argument("--solver", default="cg", choices=["cg", "eigen"])
ap.add_argument("--rank", type=int, default=64)
a = ap.parse_args()

t0 = time.time()
g, pos = G.sbm_split(n=a.n, seed=0)
t_graph = time.time() - t0
lam = kz.spectral_norm(g)
idx = kz.GraphIndex(g, 0.5 / lam, spectral_norm=lam)
t_index = 0.0
if a.solver == "eigen":  # the anchor solves start from the eigen-form low-rank term
    t0 = time.time()
    idx = kz.EigenIndex(idx, a.rank)
    t_index = time.time() - t0
# queries: endpoints of held-out pairs (nodes with positive partners), seeded
cand = np.unique(pos.ravel())
qs = G.sample_queries(cand, min(a.queries, cand.size), seed=0)
torch.cuda.synchronize()
t = time.time()
preds = kz.sparse_katz_batch(idx, qs, a.s)
torch.cuda.synchronize()
dt = time.time() - t
partners = {}
for u, v in pos:
    partners.setdefault(int(u), set()).add(int(v))
    partners.setdefault(int(v), set()).add(int(u))
rec = [len({c for c, _ in p.candidates} & partners[int(p.query)]) / len(partners[int(p.query)]) for p in preds]
out = {"solver": a.solver, "rank": a.rank if a.solver == "eigen" else None, "index_s": round(t_index, 2),
       "n": g.n, "nnz": g.nnz, "lambda": lam, "queries": len(qs), "s": a.s, "T": a.s + 1,
       "seconds": round(dt, 2), "queries_per_s": round(len(qs) / dt, 1), "graph_build_s": round(t_graph, 1),
       "recall_at_s_mean": round(float(np.mean(rec)), 4)}
if a.check:
    from oracle import katz_oracle as O

    am = O.csr_matrix(g.row_offsets, g.col_indices, g.n)
    beta = idx.alpha
    solve = lambda i: O.query_cg_csr(am, beta, int(i), tol=1e-10)[0]  # noqa: E731
    nbrs = lambda i: am.indices[am.indptr[i] : am.indptr[i + 1]]  # noqa: E731
    ok = 0
    t = time.time()
    for j in range(a.check):
        q = int(qs[j])
        want = O.sparse_katz(solve, nbrs, g.original_ids, g.internal_id(q), a.s)
        got = preds[j].candidates
        wc = dict(want)
        same_set = sorted(c for c, _ in got) == sorted(c for c, _ in want)
        corr_ok = all(abs(r - wc[c]) <= 1e-9 for c, r in got if c in wc)
        order_ok = all(c == w or abs(wc[c] - wc[w]) < 1e-9 for (c, _), (w, _) in zip(got, want))
        ok += int(same_set and corr_ok and order_ok)
    out["oracle_checked"] = a.check
    out["oracle_match"] = ok
    out["oracle_seconds_per_query"] = round((time.time() - t) / a.check, 1)
print(json.dumps(out))
